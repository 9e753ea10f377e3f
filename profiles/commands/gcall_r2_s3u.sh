# per-subdomain chunk rule: fraction of the window estimate a subdomain's chain may take (DDPMA_CHUNK_ADAPT_F)
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
for f in 0.6 0.4 0.3 0.2 0.9; do
DDPMA_CHUNK_ADAPT_F=$f timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_u_f$f.json 2> $O/bench_u_f$f.err
done
DDPMA_CHUNK_ADAPT_F=0.3 DDPMA_TIMELINE=1 timeout 300 python tools/profile_window.py C3 5 > $O/tl_u_f0.3.log 2>&1
echo done
