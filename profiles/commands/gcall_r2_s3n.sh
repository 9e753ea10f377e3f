# per-subdomain (critical-path-aware) chunk sizes vs fixed chunk sizes
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 --timeout-method=thread > $O/pytest_n.log 2>&1; echo pytest_exit=$? >> $O/pytest_n.log
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_n_adapt8.json 2> $O/bench_n_adapt8.err
DDPMA_CHUNK=6 timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_n_adapt6.json 2> $O/bench_n_adapt6.err
DDPMA_CHUNK=12 timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_n_adapt12.json 2> $O/bench_n_adapt12.err
for c in 3 4 5 6 8; do
DDPMA_CHUNK_ADAPT=0 DDPMA_CHUNK=$c timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_n_fixed$c.json 2> $O/bench_n_fixed$c.err
done
DDPMA_TIMELINE=1 timeout 300 python tools/profile_window.py C3 5 > $O/tl_adapt.log 2>&1
echo done
