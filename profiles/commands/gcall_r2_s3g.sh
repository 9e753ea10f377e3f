# barrier-merged build: parity subset + C3 bench; 4- and 2-CTA register variants
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
V=$PWD/paper_2006_14602_b200/variants
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 --timeout-method=thread > $O/pytest_g.log 2>&1; echo pytest_exit=$? >> $O/pytest_g.log
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_g_c3_b3.json 2> $O/bench_g_c3_b3.err
DDPMA_LIB=$V/libddpma_b4.so timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_g_c3_b4.json 2> $O/bench_g_c3_b4.err
DDPMA_LIB=$V/libddpma_b2.so timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_g_c3_b2.json 2> $O/bench_g_c3_b2.err
DDPMA_LIB=$V/libddpma_b4.so DDPMA_CHUNK=6 timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_g_c3_b4_c6.json 2> $O/bench_g_c3_b4_c6.err
DDPMA_LIB=$V/libddpma_b4.so DDPMA_CHUNK=12 timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_g_c3_b4_c12.json 2> $O/bench_g_c3_b4_c12.err
echo done
