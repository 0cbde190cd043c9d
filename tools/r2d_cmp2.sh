#!/bin/bash
t() { python tools/prof_step.py --config $1 --rows $2 --reps 3 | tail -1; }
for v in "$@"; do
  if [ "$v" = base ]; then unset AP_LIB_PATH; else export AP_LIB_PATH=tools/exp/$v/libalignplot_b200.so; fi
  echo "=== $v"
  echo "C4 dual K=2: $(AP_SHAPE2=16,4,2,0,1 t C4 16384)"
  echo "C4 dual K=1: $(AP_SHAPE2=16,4,1,0,1 t C4 16384)"
done
