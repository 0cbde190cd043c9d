#!/bin/bash
# Round measurement bundle (run under gpurun):  tools/profile_round.sh r01
#   1. bench.py default (C2) plain run            -> gpurun_out/$R/bench_C2.json
#   2. ncu launch list of the same command         -> gpurun_out/$R/launches_C2.csv
#   3. ncu --set full of the top kernel (C2 rows)  -> gpurun_out/$R/prof_C2.ncu-rep
#   4. other configs' bench lines                  -> gpurun_out/$R/bench_C{1,3,4}.json
R=${1:-r01}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/plain_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/prof_step.py --config C2 --rows 16285 --reps 1 > $O/prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:comb -c 1 -o $O/prof_C2 \
      python tools/prof_step.py --config C2 --rows 16285 --reps 1 > $O/ncu_full.log 2>&1
for c in C1 C3 C4; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
ls -la $O
