"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv
import sys


def main(path, top=25):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    agg = {}
    for r in rows:
        name = r[4].split("(")[0][:70]
        t = float(r[-1].replace(",", "")) / 1000.0
        a = agg.setdefault(name, [0.0, 0])
        a[0] += t
        a[1] += 1
    total = sum(v[0] for v in agg.values())
    print(f"{'us total':>10} {'n':>5} {'us/launch':>10}  kernel   ({path}, {total:.1f} us)")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{v[0]:10.1f} {v[1]:5d} {v[0] / v[1]:10.2f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
