set -x
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/gpu_profile_round.sh
timeout 600 python tools/bench_configs.py > gpurun_out/configs.jsonl 2>/dev/null
