#!/bin/bash
# Rebuild the library here (cross-compile) and refuse to continue if nvcc reported errors.
cd "$(dirname "$0")/.." || exit 1
out=$(timeout 900 python -c "import paper_2412_15840_b200.build as b; b.build(verbose=False)" 2>&1)
if echo "$out" | grep -q "error"; then
  echo "$out" | grep error | head -20
  echo "BUILD FAILED"
  exit 1
fi
echo "build ok"
