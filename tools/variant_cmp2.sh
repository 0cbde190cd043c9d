#!/bin/bash
# Compare engine builds on the GPU with device-API kernel timings (tools/prof_step.py):
#   tools/variant_cmp2.sh "C3:8192 C5:16384" base v1 ...
CFGS=$1; shift
for v in "$@"; do
  if [ "$v" = base ]; then unset AP_LIB_PATH; else export AP_LIB_PATH=tools/exp/$v/libalignplot_b200.so; fi
  r=$(python -m pytest tests/test_gpu_parity.py -x -q -k "(reference_grids or random or acceptance or threshold) and not full_size and not c5_full" 2>&1 | tail -1)
  echo "$v parity: $r"
  for cr in $CFGS; do
    c=${cr%%:*}; n=${cr##*:}
    python tools/prof_step.py --config $c --rows $n --reps ${REPS:-4} | tail -1 | sed "s/^/  $v /"
  done
done
