mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_smooth.py tests/test_arc.py -m gpu -q -s > gpurun_out/pytest_smooth.log 2>&1; echo exit=$? >> gpurun_out/pytest_smooth.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/smoke.log
