# tail chunk size scaled with the number of subdomains left (DDPMA_TAIL_SMOOTH): timed windows + e2e, A/B
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 --timeout-method=thread > $O/pytest_t.log 2>&1; echo pytest_exit=$? >> $O/pytest_t.log
timeout 400 python bench.py --no-cpu --steps 3 --warmup 3 > $O/bench_t_smooth.json 2> $O/bench_t_smooth.err
DDPMA_TAIL_SMOOTH=0 timeout 400 python bench.py --no-cpu --steps 3 --warmup 3 > $O/bench_t_plain.json 2> $O/bench_t_plain.err
timeout 400 python bench.py --no-cpu --steps 3 --warmup 3 > $O/bench_t_smooth2.json 2> $O/bench_t_smooth2.err
timeout 200 python bench.py --config C1 --until-tol 1e-6 > $O/ttc_t_c1.json 2> $O/ttc_t_c1.err
DDPMA_TIMELINE=1 timeout 300 python tools/profile_window.py C3 1 > $O/tl_t.log 2>&1
echo done
