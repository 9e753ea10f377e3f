# b3 (80-register, 3 CTAs/SM) variants: P and D benches, proxy-fence A/B, ncu --set full of one C3 window (k_windowP), 3D first windows.
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
V=$PWD/paper_2006_14602_b200/variants
DDPMA_LIB=$V/libddpma_b3.so DDPMA_KERNEL=P timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_P_b3.json 2> $O/bench_P_b3.err
DDPMA_LIB=$V/libddpma_b3.so DDPMA_KERNEL=P DDPMA_NO_PROXY_FENCE=1 timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_P_b3_nofence.json 2> $O/bench_P_b3_nofence.err
DDPMA_LIB=$V/libddpma_b3.so DDPMA_KERNEL=D timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_D_b3.json 2> $O/bench_D_b3.err
DDPMA_LIB=$V/libddpma_b3n3.so DDPMA_KERNEL=D timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_D_b3n3.json 2> $O/bench_D_b3n3.err
DDPMA_KERNEL=P timeout 300 python bench.py --config C4 --no-cpu --no-e2e --steps 2 --warmup 1 > $O/bench_c4_w23.json 2> $O/bench_c4_w23.err
DDPMA_KERNEL=P timeout 600 python bench.py --config C5 --no-cpu --no-e2e --steps 2 --warmup 1 > $O/bench_c5_w23.json 2> $O/bench_c5_w23.err
export DDPMA_LIB=$V/libddpma_b3.so DDPMA_KERNEL=P
timeout 300 python tools/profile_window.py C3 2 > $O/plainP.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_windowP -s 2 -c 1 \
  -o $O/r2_c3_windowP_b3 python tools/profile_window.py C3 2 > $O/ncuP.log 2>&1
echo done
