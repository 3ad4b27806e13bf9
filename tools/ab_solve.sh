#!/bin/bash
# A/B of solve variants: tools/ab_solve.sh "VAR=a VAR2=b" "VAR=c" ...  (each arg = env assignments)
cd "$(dirname "$0")/.."
for spec in "$@"; do
  echo "== $spec"
  for c in ${AB_CONFIGS:-c1 c2 c3}; do
    env $spec timeout 120 python tools/profile_step.py --config $c --reps ${AB_REPS:-3} 2>&1 | head -1
  done
done
