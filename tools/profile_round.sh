#!/bin/bash
# Round measurement bundle (run under gpurun):  tools/profile_round.sh r01
#   bench lines (all five configs, CPU reference sample beside each), the reference arm,
#   the ncu launch list of the default bench (C2), and ncu --set full of the comb kernel
#   per config (full grid for C1/C2, a row block for C3-C5)            -> gpurun_out/$R/
R=${1:-r01}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_C2_reference.json 2> $O/bench_C2_reference.err
python bench.py --config C1 > $O/bench_C1.json 2> $O/bench_C1.err
python bench.py --config C3 --steps 5 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
python bench.py --config C4 --steps 3 --warmup 3 > $O/bench_C4.json 2> $O/bench_C4.err
python bench.py --config C5 --steps 1 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/plain_small.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
for cr in C1:0 C2:0 C3:8192 C4:4096 C5:512; do
  c=${cr%%:*}; n=${cr##*:}
  python tools/prof_step.py --config $c --rows $n --reps 1 > $O/prof_$c.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:comb -c 1 -o $O/prof_$c \
        python tools/prof_step.py --config $c --rows $n --reps 1 > $O/ncu_full_$c.log 2>&1
  # summarise on the box (gpurun brings back <= 64 MiB); keep only the C2 report
  python tools/ncu_summary.py $O/prof_$c.ncu-rep --top 12 > $O/ncu_summary_$c.txt 2>&1
  [ $c = C2 ] || rm -f $O/prof_$c.ncu-rep
done
python tools/d2h_bw.py > $O/d2h_bw.txt 2>&1
ls -la $O
