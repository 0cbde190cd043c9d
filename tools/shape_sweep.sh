#!/bin/bash
# Time candidate kernel shapes (AP_SHAPE="L,R,K[,xm]") on a config subset.
#   tools/shape_sweep.sh C3 8192 "8,16,2 8,16,4 16,16,2"
cfg=$1; rows=$2; shapes=$3
for s in $shapes; do
  printf "%-10s " "$s"; AP_SHAPE=$s python tools/prof_step.py --config $cfg --rows $rows --reps 2 | tail -1
done
