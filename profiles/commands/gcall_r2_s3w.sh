# 3D window kernel at 2 CTAs/SM (128 registers) vs 3 CTAs/SM (80 registers)
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
V=$PWD/paper_2006_14602_b200/variants
for v in base m3b2; do
L=""; [ $v != base ] && L=$V/libddpma_$v.so
DDPMA_LIB=$L timeout 400 python bench.py --config C5 --dtau 2e-6 --no-cpu --no-e2e --steps 2 --warmup 3 > $O/bench_w_c5_$v.json 2> $O/bench_w_c5_$v.err
DDPMA_LIB=$L timeout 300 python bench.py --config C4 --dtau 1e-4 --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_w_c4_$v.json 2> $O/bench_w_c4_$v.err
done
echo done
