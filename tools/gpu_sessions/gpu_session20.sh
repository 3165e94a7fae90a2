# superpass default: full GPU suite + smoke + bench
set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/b20.json 2> gpurun_out/b20.err; cat gpurun_out/b20.json; tail -3 gpurun_out/b20.err
