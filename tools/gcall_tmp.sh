timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench_v3.json 2> gpurun_out/bench_v3.err
DDPMA_CHUNK=16 timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench_v3_c16.json 2> gpurun_out/bench_v3_c16.err
