#!/bin/bash
# ncu --set full of one config's comb kernel under shape overrides:
#   tools/prof_shape.sh <tag> <config:rows> "ENV=VAL ..." [more env sets]
R=$1; cr=$2; shift 2; O=gpurun_out/$R; mkdir -p $O
c=${cr%%:*}; n=${cr##*:}; i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs python tools/prof_step.py --config $c --rows $n --reps 2 > $O/prof_$i.log 2>&1 && \
    env $envs ncu --set full --clock-control none --import-source on -k regex:comb -c 1 -o $O/prof_$i \
        python tools/prof_step.py --config $c --rows $n --reps 1 > $O/ncu_full_$i.log 2>&1
  (echo "# $envs"; tail -1 $O/prof_$i.log; python tools/ncu_summary.py $O/prof_$i.ncu-rep --top 12) > $O/ncu_summary_$i.txt 2>&1
  rm -f $O/prof_$i.ncu-rep
done
