#!/bin/bash
# A/B timing of variant libraries on one case (run under gpurun).
# Usage: bash scripts/ab_run.sh "<env for timeline.py>" name1 name2 ...   (name "base" = the in-tree library)
ENVS=$1; shift
mkdir -p gpurun_out
for n in "$@"; do
  if [ "$n" = base ]; then L=""; else L="$PWD/build_exp/libmp_$n.so"; fi
  echo "== $n"
  env $ENVS MP_B200_LIB=$L python scripts/timeline.py 2>&1 | grep -v "^  info"
done
