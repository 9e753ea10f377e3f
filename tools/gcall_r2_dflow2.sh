mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/smoke.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -rA -s -k "c1_prefix or baseline_window or deterministic or one_by_one or c1_default_prefix or rerun or uniform" > gpurun_out/pytest_dflow.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_dflow.log
for v in D P; do
DDPMA_KERNEL=$v timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err
DDPMA_KERNEL=$v DDPMA_NO_PROXY_FENCE=1 timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/bench_${v}nf.json 2> gpurun_out/bench_${v}nf.err
done
echo done
