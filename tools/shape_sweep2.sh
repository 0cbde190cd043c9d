#!/bin/bash
# Time r=2 kernel shapes (AP_SHAPE2="L,RR,K") on a config subset.
cfg=$1; rows=$2; shapes=$3
for s in $shapes; do
  printf "%-10s " "$s"; AP_SHAPE2=$s python tools/prof_step.py --config $cfg --rows $rows --reps 2 | tail -1
done
