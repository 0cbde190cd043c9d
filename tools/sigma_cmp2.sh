#!/bin/bash
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dual" 2>&1 | tail -2
for sw in "20 128" "20 256" "60 64" "60 128" "40 128" "120 64" "20 64" "4 128" "30 512"; do
  set -- $sw
  python tools/sigma_step.py --sigma $1 --w $2 | tail -1
done
