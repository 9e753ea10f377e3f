# claim-ahead build: GPU parity tests + C3/C4/C5 benches
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread > $O/pytest_h.log 2>&1; echo pytest_exit=$? >> $O/pytest_h.log
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_h_c3.json 2> $O/bench_h_c3.err
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 --profile stable > $O/bench_h_c3_stable.json 2> $O/bench_h_c3_stable.err
timeout 300 python bench.py --config C4 --dtau 1e-4 --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_h_c4.json 2> $O/bench_h_c4.err
timeout 400 python bench.py --config C5 --dtau 2e-6 --no-cpu --no-e2e --steps 2 --warmup 3 > $O/bench_h_c5.json 2> $O/bench_h_c5.err
echo done
