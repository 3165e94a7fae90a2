# flakiness check: the concurrency-heavy tests (L2-blocked step, sharded) three times
for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_sharded.py -m gpu -q -x -k "super or bitwise or n30 or sharded" -p no:randomly 2>&1 | tail -1; done
