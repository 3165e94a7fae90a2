set -x
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for rb in 3 4; do for sp in 1 0; do for cp in 1 2; do
python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --row-bits $rb --step-spanning $sp --ctas-per-sm $cp > gpurun_out/bench_rb${rb}_sp${sp}_c${cp}.json 2>&1
done; done; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:qaa_pass_kernel -s 6 -c 3 -o gpurun_out/prof_pass python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
