# extreme-value parity of the two-node log-equidistribution path
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rA -s -k "extreme" --timeout 300 --timeout-method=thread > gpurun_out/pytest_z.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_z.log
echo done
