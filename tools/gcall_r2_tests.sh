mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA -s --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
