#!/bin/bash
for sw in "20 128" "20 256" "60 64" "60 128" "40 128" "120 64"; do
  set -- $sw
  echo "== sigma $1 w $2"
  AP_NO_DUAL=1 python tools/sigma_step.py --sigma $1 --w $2 | tail -1
  for s in 4,32,1 8,16,2 16,8,2 8,8,2 8,32,2 16,16,1 4,16,2 32,8,2; do
    AP_DUAL=1 AP_SHAPE=$s,0,-1,1 python tools/sigma_step.py --sigma $1 --w $2 2>/dev/null | tail -1 | grep combd
  done
done
true
