python tools/kernel_times.py distilbert 5 2>&1 | grep -v Warn | sed -n 2,9p
GG_NO_PDL=1 python tools/kernel_times.py distilbert 5 2>&1 | grep -v Warn | sed -n 2,9p
