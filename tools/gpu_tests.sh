#!/bin/bash
# Run each GPU test file under its own timeout so a hang is localized (used with gpurun).
for f in ${@:-tests/test_*.py}; do
  echo "== $f"
  timeout ${GG_TEST_TIMEOUT:-240} python -m pytest "$f" -m gpu -q -x -v 2>&1 | grep -E "PASSED|FAILED|ERROR|passed|failed|Error|error" | tail -40
  echo "rc=$?"
done
