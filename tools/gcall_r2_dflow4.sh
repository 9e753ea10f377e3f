mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rA -s -k "c1_prefix or baseline_window or deterministic or one_by_one or c1_default_prefix or rerun or uniform" > gpurun_out/pytest_dflow.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_dflow.log
timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_D.json 2> gpurun_out/bench_D.err
DDPMA_CHUNK=16 timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_D16.json 2> gpurun_out/bench_D16.err
DDPMA_TIMELINE=1 timeout 300 python tools/profile_window.py C3 3 > gpurun_out/tl_D.log 2>&1
echo done
