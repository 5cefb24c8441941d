#!/bin/bash
# ncu evidence for profiles/ (run under gpurun; single GPU; never a bench number).
#   launch lists: per-kernel device time + DRAM bytes of serving steps (ResNet-18,
#                 DistilBERT) and of one full-batch forward each
#   full captures: the dominant conv / GEMM / admission kernels (details + raw metrics)
set -u
OUT=${1:-gpurun_out/prof}
mkdir -p "$OUT"
NCU="ncu --clock-control none"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 300 $NCU --metrics $M --csv --log-file "$OUT/resnet18_step_launches.csv" python tools/serve_once.py resnet18 3 > /dev/null 2>&1
timeout 300 $NCU --metrics $M --csv --log-file "$OUT/distilbert_step_launches.csv" python tools/serve_once.py distilbert 2 > /dev/null 2>&1
timeout 300 $NCU --metrics $M --csv --log-file "$OUT/resnet18_forward_launches.csv" python tools/forward_once.py resnet18 1 > /dev/null 2>&1
timeout 300 $NCU --metrics $M --csv --log-file "$OUT/distilbert_forward_launches.csv" python tools/forward_once.py distilbert 1 > /dev/null 2>&1
# one full capture per dominant kernel (a forward's instance)
timeout 300 $NCU --set full --import-source on -k regex:conv_span_pair -s 3 -c 1 \
  -o "$OUT/resnet18_layer3_span_pair" python tools/forward_once.py resnet18 1 > /dev/null 2>&1
timeout 300 $NCU --set full --import-source on -k regex:conv_span_px2 -s 1 -c 1 \
  -o "$OUT/resnet18_layer1_span" python tools/forward_once.py resnet18 1 > /dev/null 2>&1
timeout 300 $NCU --set full --import-source on -k regex:gemm_bf16_pair -s 2 -c 1 \
  -o "$OUT/distilbert_ffn_up_gemm_pair" python tools/forward_once.py distilbert 1 > /dev/null 2>&1
timeout 300 $NCU --set full --import-source on -k regex:conv_bf16_tcgen05 -s 1 -c 1 \
  -o "$OUT/resnet18_stride2_conv_ds" python tools/forward_once.py resnet18 1 > /dev/null 2>&1
timeout 300 $NCU --set full --import-source on -k regex:attention -s 1 -c 1 \
  -o "$OUT/distilbert_attention" python tools/forward_once.py distilbert 1 > /dev/null 2>&1
timeout 300 $NCU --set full --import-source on -k regex:stem_pool_span -s 0 -c 1 \
  -o "$OUT/resnet18_stem_pool" python tools/forward_once.py resnet18 1 > /dev/null 2>&1
timeout 300 $NCU --set full --import-source on -k regex:cls_head_kernel -s 0 -c 1 \
  -o "$OUT/distilbert_cls_head" python tools/forward_once.py distilbert 1 > /dev/null 2>&1
timeout 300 $NCU --set full --import-source on -k regex:fallback_kernel -s 1 -c 1 \
  -o "$OUT/resnet18_fallback_cluster" python tools/serve_once.py resnet18 3 > /dev/null 2>&1
GG_PROBE_EAGER=1 timeout 300 $NCU --set full --import-source on -k regex:admit_small_kernel -s 1 -c 1 \
  -o "$OUT/k1_admit_2p26" python tools/kernel_probe.py k1 1 > /dev/null 2>&1
for f in "$OUT"/*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i "$f" --page details --csv > "$b.details.csv" 2>/dev/null
  ncu -i "$f" --page raw --csv > "$b.raw.csv" 2>/dev/null
done
ls -la "$OUT"
