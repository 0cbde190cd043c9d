mkdir -p gpurun_out/q
python -m pytest tests -m gpu -x -q > gpurun_out/q/tests.log 2>&1; tail -3 gpurun_out/q/tests.log
for c in C1 C2 C3; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:3], round(d['ms_per_step'],4), '%.3e'%d['value'])"; done
python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4', round(d['ms_per_step'],2), '%.3e'%d['value'])"
