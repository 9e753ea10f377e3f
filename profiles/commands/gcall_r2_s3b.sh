# P-kernel baseline (stage-by-stage window kernel): GPU tests, smoke, register variants; D-kernel hang probe.
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
DDPMA_KERNEL=P timeout 1200 python -m pytest tests -m gpu -q -rA --durations=15 --timeout 300 --timeout-method=thread > $O/pytest_gpu_P.log 2>&1; echo pytest_exit=$? >> $O/pytest_gpu_P.log
DDPMA_KERNEL=P timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_P.log 2>&1; echo smoke_exit=$? >> $O/smoke_P.log
timeout 90 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_D.log 2>&1; echo smoke_exit=$? >> $O/smoke_D.log
for v in b3 b2; do
DDPMA_LIB=$PWD/paper_2006_14602_b200/variants/libddpma_$v.so DDPMA_KERNEL=P timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_P_$v.json 2> $O/bench_P_$v.err
done
DDPMA_KERNEL=P timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_P_b4.json 2> $O/bench_P_b4.err
echo done
