for n in 24 26 28 30; do for sup in 3 7 1; do for K in 1 2 5; do
echo "== n=$n sup=$sup K=$K"; timeout 40 python tools/diag_super.py $n $sup $K 2>&1 | tail -2
done; done; done
