# tail knobs on the adaptive-chunk build (information only)
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_p_base.json 2> $O/bench_p_base.err
DDPMA_TAIL_N=8 timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_p_tn8.json 2> $O/bench_p_tn8.err
DDPMA_TAIL_N=32 timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_p_tn32.json 2> $O/bench_p_tn32.err
DDPMA_CHUNK_TAIL=1 timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_p_ct1.json 2> $O/bench_p_ct1.err
DDPMA_CHUNK_TAIL=3 timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_p_ct3.json 2> $O/bench_p_ct3.err
DDPMA_CHUNK_TAIL=4 timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_p_ct4.json 2> $O/bench_p_ct4.err
timeout 400 python bench.py --no-cpu --steps 3 --warmup 3 > $O/bench_p_e2e.json 2> $O/bench_p_e2e.err
DDPMA_CHUNK_TAIL=1 timeout 400 python bench.py --no-cpu --steps 3 --warmup 3 > $O/bench_p_e2e_ct1.json 2> $O/bench_p_e2e_ct1.err
echo done
