#!/bin/bash
t() { python tools/prof_step.py --config $1 --rows $2 --reps 3 | tail -1; }
for v in "$@"; do
  if [ "$v" = base ]; then unset AP_LIB_PATH; else export AP_LIB_PATH=tools/exp/$v/libalignplot_b200.so; fi
  echo "=== $v"
  python -m pytest tests/test_gpu_parity.py -x -q -k "forced_r2_shapes or acceptance" 2>&1 | tail -1
  echo "C4: $(t C4 16384)"
  echo "C2: $(t C2 0)"
done
