# integer-decomposition fastlog: parity subset + C3 bench; compute-sanitizer memcheck on C1 + T3 solves
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 --timeout-method=thread > $O/pytest_i.log 2>&1; echo pytest_exit=$? >> $O/pytest_i.log
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_i_c3.json 2> $O/bench_i_c3.err
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 --profile stable > $O/bench_i_c3_stable.json 2> $O/bench_i_c3_stable.err
timeout 300 python tools/sanitize_case.py 3 2 > $O/san_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_case.py 3 2 > $O/san_memcheck.log 2>&1
echo san_exit=$? >> $O/san_memcheck.log
echo done
