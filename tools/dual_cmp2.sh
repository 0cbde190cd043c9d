#!/bin/bash
# Dual-pair kernel variants: parity subset on the default build, then kernel timings per variant.
python -m pytest tests/test_gpu_parity.py -x -q -k "reference_grids or random or acceptance or threshold" 2>&1 | tail -2
t() { python tools/prof_step.py --config $1 --rows $2 --reps 3 | tail -1; }
for v in "$@"; do
  if [ "$v" = base ]; then unset AP_LIB_PATH; else export AP_LIB_PATH=tools/exp/$v/libalignplot_b200.so; fi
  echo "=== $v"
  for s in 4,32,2 8,16,2 4,32,1; do echo "C3 dual $s: $(AP_SHAPE=$s,0,-1,1 t C3 0)"; done
  for s in 8,32,2 16,16,2 8,32,1; do echo "C5 dual $s: $(AP_SHAPE=$s,0,-1,1 t C5 8192)"; done
done
