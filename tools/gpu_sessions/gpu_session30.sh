# plan choice vs size: L2-blocked step on/off for n = 20..30
for n in 20 21 22 23 24 25 26 27 28 29 30; do for m in 1 0; do timeout 120 python tools/diag_super2.py $m 50 $n 2>&1 | sed "s/^/n=$n /"; done; done
