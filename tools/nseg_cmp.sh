#!/bin/bash
t() { python tools/prof_step.py --config $1 --rows $2 --reps 3 | tail -1; }
for n in 0 3 4 5 6 8 12 16; do
  if [ $n = 0 ]; then unset AP_NSEG; else export AP_NSEG=$n; fi
  echo "C3 nseg=$n: $(t C3 0)"
done
unset AP_NSEG
for tw in 0.5 1 2; do echo "C3 tail_waves=$tw: $(AP_TAIL_WAVES=$tw t C3 0)"; done
echo "C3 no tail split: $(AP_TAIL_SPLIT=1 t C3 0)"
echo "C3 tail split 4: $(AP_TAIL_SPLIT=4 t C3 0)"
