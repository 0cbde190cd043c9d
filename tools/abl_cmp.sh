#!/bin/bash
# Timing-only comparison of engine builds (no parity run: ablation builds give wrong results):
#   tools/abl_cmp.sh "C3:8192 C5:8192" base v1 ...
CFGS=$1; shift
for v in "$@"; do
  if [ "$v" = base ]; then unset AP_LIB_PATH; else export AP_LIB_PATH=tools/exp/$v/libalignplot_b200.so; fi
  for cr in $CFGS; do
    c=${cr%%:*}; n=${cr##*:}
    python tools/prof_step.py --config $c --rows $n --reps ${REPS:-4} | tail -1 | sed "s/^/  $v /"
  done
done
