set -x
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for k in 1 0; do
timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --no-e2e --kernel $k > gpurun_out/b3_k${k}.json 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches3.csv python bench.py --steps 1 --warmup 1 --chunk 10 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qaa_pass_tma -s 3 -c 3 -o gpurun_out/prof_tma python bench.py --steps 1 --warmup 0 --chunk 6 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full3.log 2>&1
