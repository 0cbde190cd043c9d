#!/bin/bash
# Dual-pair kernel: parity subset, then kernel timings of shapes against the single-pair kernel.
python -m pytest tests/test_gpu_parity.py -x -q -k "reference_grids or random or acceptance or threshold" 2>&1 | tail -3
t() { python tools/prof_step.py --config $1 --rows $2 --reps 3 | tail -1; }
echo "== C3"; AP_NO_DUAL=1 t C3 0
for s in 4,32,2 4,32,1 8,16,2 8,16,1; do echo "dual $s"; AP_SHAPE=$s,0,-1,1 t C3 0; AP_SHAPE=$s,0,0,1 t C3 0; done
echo "== C5"; AP_NO_DUAL=1 t C5 8192
for s in 8,32,2 8,32,1 16,16,2 16,16,1; do echo "dual $s"; AP_SHAPE=$s,0,-1,1 t C5 8192; AP_SHAPE=$s,0,0,1 t C5 8192; done
echo "== C1"; AP_NO_DUAL=1 t C1 0
for s in 8,8,2 8,8,1 4,16,2; do echo "dual $s"; AP_SHAPE=$s,0,-1,1 t C1 0; done
