#!/bin/bash
# Round-2 measurement bundle (run under gpurun):  tools/profile_r02.sh <tag> [configs]
#   ncu launch list of the default bench (C4), and ncu --set full of the comb kernel per
#   config (full plot for C1-C4, a row block for C5) with summaries -> gpurun_out/<tag>/
R=${1:-r02}
CFGS=${2:-"C4:0 C3:0 C5:32768 C2:0 C1:0"}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/plain_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/ncu_launch_summary.py $O/launches_C4.csv "python bench.py --steps 2 --warmup 1 --no-cpu-baseline (C4)" \
  > $O/launches_C4_summary.txt 2>&1
for cr in $CFGS; do
  c=${cr%%:*}; n=${cr##*:}
  python tools/prof_step.py --config $c --rows $n --reps 1 > $O/prof_$c.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:comb -c 1 -o $O/prof_$c \
        python tools/prof_step.py --config $c --rows $n --reps 1 > $O/ncu_full_$c.log 2>&1
  python tools/ncu_summary.py $O/prof_$c.ncu-rep --top 16 > $O/ncu_summary_$c.txt 2>&1
  [ $c = C4 ] || rm -f $O/prof_$c.ncu-rep
done
ls -la $O
