# first tile of a chunk issued by the claiming thread right after the claim: parity + benches
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread > $O/pytest_v.log 2>&1; echo pytest_exit=$? >> $O/pytest_v.log
timeout 400 python bench.py --no-cpu --steps 3 --warmup 3 > $O/bench_v_c3.json 2> $O/bench_v_c3.err
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_v_c3_b.json 2> $O/bench_v_c3_b.err
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_v_c3_c.json 2> $O/bench_v_c3_c.err
echo done
