#!/bin/bash
# Round bench bundle (run under gpurun):  tools/bench_round.sh <tag>
#   bench.py lines for all five configs (CPU reference sample + parity beside each), the
#   reference arm of the default config, and the peak microbenchmarks -> gpurun_out/<tag>/
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
nproc > $O/nproc.txt
python bench.py --steps 20 --warmup 5 > $O/bench_C4.json 2> $O/bench_C4.err
python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_C4_reference.json 2> $O/bench_C4_reference.err
python bench.py --config C1 --steps 20 --warmup 5 > $O/bench_C1.json 2> $O/bench_C1.err
python bench.py --config C2 --steps 20 --warmup 5 > $O/bench_C2.json 2> $O/bench_C2.err
python bench.py --config C3 --steps 10 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
python bench.py --config C5 --steps 2 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o $O/lds_peak.bin tools/lds_peak.cu && $O/lds_peak.bin > $O/lds_peak.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o $O/int_peak.bin tools/int_peak.cu && $O/int_peak.bin > $O/int_peak.txt 2>&1
rm -f $O/*.bin
ls -la $O
