#!/bin/bash
# Compare engine builds on the GPU: tools/variant_cmp.sh "C3 C1" base kh1 ...
# (base = the in-tree build; others = tools/exp/<name>/libalignplot_b200.so)
CFGS=$1; shift
mkdir -p gpurun_out/vc
for v in "$@"; do
  if [ "$v" = base ]; then unset AP_LIB_PATH; else export AP_LIB_PATH=tools/exp/$v/libalignplot_b200.so; fi
  r=$(python -m pytest tests/test_gpu_parity.py -x -q -k "(reference_grids or random or acceptance or threshold) and not full_size and not c5_full" 2>&1 | tail -1)
  echo "$v parity: $r"
  for c in $CFGS; do
    python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  $v', '$c', round(d['ms_per_step'],4), '%.4e'%d['value'])"
  done
done
