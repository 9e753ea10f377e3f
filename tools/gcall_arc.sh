mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_arc.py -m gpu -q -s > gpurun_out/pytest_arc.log 2>&1; echo arc_exit=$? >> gpurun_out/pytest_arc.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
