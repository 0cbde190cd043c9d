#!/bin/bash
# ncu --set full of the comb kernel for a config:  tools/prof_dual.sh <tag> "C3:0 C5:8192"
R=$1; CFGS=$2; O=gpurun_out/$R; mkdir -p $O
for cr in $CFGS; do
  c=${cr%%:*}; n=${cr##*:}
  python tools/prof_step.py --config $c --rows $n --reps 1 > $O/prof_$c.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:comb -c 1 -o $O/prof_$c \
        python tools/prof_step.py --config $c --rows $n --reps 1 > $O/ncu_full_$c.log 2>&1
  python tools/ncu_summary.py $O/prof_$c.ncu-rep --top 24 > $O/ncu_summary_$c.txt 2>&1
done
