#!/bin/bash
# quick A/B of TC screen configurations on the c2 shape (GPU box)
for cfg in "256 2 8" "256 1 8" "128 2 8" "128 1 8" "256 2 2" "128 2 3"; do
  set -- $cfg
  echo "BN=$1 ABUFS=$2 STAGES=$3"
  FTK_TC_BN=$1 FTK_TC_ABUFS=$2 FTK_TC_STAGES=$3 timeout 120 python tools/prof_assign.py --variant tc --reps 2 | tail -1
done
