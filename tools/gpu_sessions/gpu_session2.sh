set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for cp in 1 2; do for rb in 3 4; do
python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --row-bits $rb --ctas-per-sm $cp > gpurun_out/b2_rb${rb}_c${cp}.json 2>&1
done; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 1 --warmup 1 --chunk 10 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:qaa_pass_fast -s 3 -c 3 -o gpurun_out/prof_fast python bench.py --steps 1 --warmup 0 --chunk 6 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full2.log 2>&1
