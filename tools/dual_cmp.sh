#!/bin/bash
# Dual-pair kernel variants: kernel timings per variant (shape lists in SH3 / SH5).
t() { python tools/prof_step.py --config $1 --rows $2 --reps 3 | tail -1; }
for v in "$@"; do
  if [ "$v" = base ]; then unset AP_LIB_PATH; else export AP_LIB_PATH=tools/exp/$v/libalignplot_b200.so; fi
  echo "=== $v"
  for s in ${SH3:-4,32,2 4,32,1 8,16,2 8,16,1}; do echo "C3 dual $s: $(AP_SHAPE=$s,0,-1,1 t C3 0)"; done
  for s in ${SH5:-8,32,2 8,32,1 16,16,2 16,16,1}; do echo "C5 dual $s: $(AP_SHAPE=$s,0,-1,1 t C5 8192)"; done
done
