set -x
timeout 300 python tools/bench_configs.py > gpurun_out/configs.jsonl 2>&1
timeout 300 python tools/bench_energy.py > gpurun_out/energy_F2.json 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --share-gpu --qubits 26 --steps 3 --warmup 1 --chunk 10 --no-cpu-baseline > gpurun_out/bench_share2.json 2> gpurun_out/bench_share2.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --share-gpu --qubits 26 --steps 3 --warmup 1 --chunk 10 --no-cpu-baseline > gpurun_out/bench_share4.json 2> gpurun_out/bench_share4.err
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "max_size or empty_instance" 2>&1 | tail -4
