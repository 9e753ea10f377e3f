mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/smoke.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rA -s -k "c1_prefix or baseline_window or deterministic or one_by_one or c1_default_prefix or rerun or uniform or t3 or c4" > gpurun_out/pytest_dflow.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_dflow.log
for v in D P; do
DDPMA_KERNEL=$v timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
done
DDPMA_TIMELINE=1 timeout 300 python tools/profile_window.py C3 3 > gpurun_out/tl_D.log 2>&1
timeout 600 python bench.py --config C5 --no-cpu --no-e2e --steps 2 --warmup 3 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 600 python bench.py --config C4 --no-cpu --no-e2e --steps 5 --warmup 3 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
echo done
