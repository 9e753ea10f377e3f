# one barrier per chunk (claim after compute, completion deferred to warp 1): parity + benches
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread > $O/pytest_s.log 2>&1; echo pytest_exit=$? >> $O/pytest_s.log
timeout 400 python bench.py --no-cpu --steps 3 --warmup 3 > $O/bench_s_c3.json 2> $O/bench_s_c3.err
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_s_c3_b.json 2> $O/bench_s_c3_b.err
timeout 400 python bench.py --config C5 --dtau 2e-6 --no-cpu --no-e2e --steps 2 --warmup 3 > $O/bench_s_c5.json 2> $O/bench_s_c5.err
timeout 300 python bench.py --config C4 --dtau 1e-4 --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_s_c4.json 2> $O/bench_s_c4.err
echo done
