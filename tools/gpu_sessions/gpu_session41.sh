for m in 1 65 1 65 1 65; do timeout 120 python tools/diag_super2.py $m 20 30; done
