#!/bin/bash
# compute-sanitizer evidence (run under gpurun, one GPU).
#   memcheck  : __graft_entry__.smoke() end to end (K1 / K2 / K3, the serving loop with
#               the fallback cluster, FIFO, gathers and publish, both forwards, the head)
#               + the fused-head and fallback tests
#   racecheck / synccheck : the controller kernels, the DistilBERT forward (pair GEMMs
#               with LayerNorm folding, attention, head) and the DistilBERT serving loop.
#               The ResNet span convolutions are listed separately (see profiles/r2/sanitizer.md).
set -u
OUT=${1:-gpurun_out/sanitize}
mkdir -p "$OUT"
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
run() {   # name tool cmd...
  local name=$1 tool=$2; shift 2
  echo "== $tool: $name" | tee -a "$OUT/summary.txt"
  timeout 1500 $CS --tool "$tool" "$@" > "$OUT/${name}_$tool.log" 2>&1
  echo "exit $?" | tee -a "$OUT/summary.txt"
  grep -E "passed|failed|ERROR SUMMARY|RACECHECK SUMMARY|smoke ok" "$OUT/${name}_$tool.log" | tail -3 | tee -a "$OUT/summary.txt"
}
run smoke memcheck python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")'
run head_fallback memcheck python -m pytest -q tests/test_distilbert_gpu.py tests/test_serving_gpu.py \
  -k "fused_head or fallback_answers_large_window"
SEL_D="logits_vs_eager and 4 or layernorm_folding or fused_head and 4"
SEL_C="literal or decide_literal or outcome_literals or utility_rows or epilogue_vs_oracle or fast_filter"
SEL_S="distilbert and not resnet and not open and True"
for tool in racecheck synccheck; do
  run controller $tool python -m pytest -q tests/test_controller_gpu.py -k "$SEL_C"
  run distilbert $tool python -m pytest -q tests/test_distilbert_gpu.py -k "$SEL_D"
  run serving_distilbert $tool python -m pytest -q tests/test_serving_gpu.py -k "$SEL_S"
  run span_conv $tool python -m pytest -q tests/test_conv_span_gpu.py -k "test_span_conv_vs_torch"
done
