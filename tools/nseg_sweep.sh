for ns in 4 5 6 8 10 12 16; do printf "nseg=%-3s " $ns; AP_NSEG=$ns python tools/prof_step.py --config C2 --rows 16285 --reps 3 | tail -1; done
for ns in 2 3 4 6; do printf "C3 nseg=%-3s " $ns; AP_NSEG=$ns python tools/prof_step.py --config C3 --rows 65409 --reps 2 | tail -1; done
