# 2D TMA ring depth 2 vs 3; bulk chunk sizes on the 80-register build
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
V=$PWD/paper_2006_14602_b200/variants
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 --timeout-method=thread > $O/pytest_m.log 2>&1; echo pytest_exit=$? >> $O/pytest_m.log
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_m_ring2.json 2> $O/bench_m_ring2.err
DDPMA_LIB=$V/libddpma_ring3.so timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_m_ring3.json 2> $O/bench_m_ring3.err
DDPMA_LIB=$V/libddpma_ring3.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 --timeout-method=thread -k "c1_prefix or baseline or uniform or rerun or c1_reference" > $O/pytest_m_ring3.log 2>&1; echo pytest_exit=$? >> $O/pytest_m_ring3.log
for c in 6 10 12; do
DDPMA_CHUNK=$c timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_m_ring2_c$c.json 2> $O/bench_m_ring2_c$c.err
DDPMA_LIB=$V/libddpma_ring3.so DDPMA_CHUNK=$c timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_m_ring3_c$c.json 2> $O/bench_m_ring3_c$c.err
done
DDPMA_LIB=$V/libddpma_ring3.so DDPMA_CHUNK_TAIL=3 timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_m_ring3_t3.json 2> $O/bench_m_ring3_t3.err
echo done
