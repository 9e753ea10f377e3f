# After the tile-only physical-face formulas (code size 19K instr per kernel): full GPU tests, smoke, C3/C4/C5 benches, D check.
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -rA --durations=10 --timeout 300 --timeout-method=thread > $O/pytest_gpu_f.log 2>&1; echo pytest_exit=$? >> $O/pytest_gpu_f.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_f.log 2>&1; echo smoke_exit=$? >> $O/smoke_f.log
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_f_c3.json 2> $O/bench_f_c3.err
DDPMA_KERNEL=D timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_f_c3_D.json 2> $O/bench_f_c3_D.err
timeout 300 python bench.py --config C4 --dtau 1e-4 --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_f_c4.json 2> $O/bench_f_c4.err
timeout 400 python bench.py --config C5 --dtau 2e-6 --no-cpu --no-e2e --steps 2 --warmup 3 > $O/bench_f_c5.json 2> $O/bench_f_c5.err
echo done
