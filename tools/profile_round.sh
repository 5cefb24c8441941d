#!/bin/bash
# ncu evidence for profiles/ (run under gpurun; single GPU; never a bench number).
#   launch lists: per-kernel device time of the serving step (ResNet-18, DistilBERT)
#   full captures: the dominant conv / GEMM / admission kernels (details + raw metrics)
set -u
OUT=${1:-gpurun_out/prof}
mkdir -p "$OUT"
NCU="ncu --clock-control none"
timeout 300 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file "$OUT/resnet18_step_launches.csv" python tools/serve_once.py resnet18 3 > /dev/null 2>&1
timeout 300 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv \
  --log-file "$OUT/distilbert_step_launches.csv" python tools/serve_once.py distilbert 2 > /dev/null 2>&1
# one full capture per dominant kernel (second step's instance)
timeout 300 $NCU --set full --import-source on -k regex:conv_span_tcgen05 -s 12 -c 1 \
  -o "$OUT/resnet18_span_conv" python tools/serve_once.py resnet18 3 > /dev/null 2>&1
timeout 300 $NCU --set full --import-source on -k regex:gemm_bf16_tcgen05 -s 30 -c 1 \
  -o "$OUT/distilbert_gemm" python tools/serve_once.py distilbert 2 > /dev/null 2>&1
GG_PROBE_EAGER=1 timeout 300 $NCU --set full --import-source on -k regex:admit_small_kernel -s 1 -c 1 \
  -o "$OUT/k1_admit_2p26" python tools/kernel_probe.py k1 1 > /dev/null 2>&1
for f in "$OUT"/*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i "$f" --page details --csv > "$b.details.csv" 2>/dev/null
  ncu -i "$f" --page raw --csv > "$b.raw.csv" 2>/dev/null
done
ls -la "$OUT"
