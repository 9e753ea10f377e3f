# 3D compute in three phases (determinants, two-node log-equidistribution, epilogues): parity + benches
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread > $O/pytest_y.log 2>&1; echo pytest_exit=$? >> $O/pytest_y.log
timeout 400 python bench.py --config C5 --dtau 2e-6 --no-cpu --no-e2e --steps 2 --warmup 3 > $O/bench_y_c5.json 2> $O/bench_y_c5.err
timeout 300 python bench.py --config C4 --dtau 1e-4 --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_y_c4.json 2> $O/bench_y_c4.err
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_y_c3.json 2> $O/bench_y_c3.err
echo done
