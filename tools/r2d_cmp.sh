#!/bin/bash
t() { python tools/prof_step.py --config $1 --rows $2 --reps 3 | tail -1; }
python -m pytest tests/test_gpu_parity.py -x -q -k "r2_dual" 2>&1 | tail -3
echo "C4 single: $(AP_NO_DUAL=1 t C4 16384)"
echo "C4 dual K=2: $(AP_SHAPE2=16,4,2,0,1 t C4 16384)"
echo "C4 dual K=1: $(AP_SHAPE2=16,4,1,0,1 t C4 16384)"
