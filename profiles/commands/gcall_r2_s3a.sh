# Round-2 re-entry baseline on a fresh B200: GPU tests, smoke, C3 bench (D and P kernels),
# C4/C5 3D benches, time-to-converged, ncu launch list + --set full of one C3 window.
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=15 > $O/pytest_gpu.log 2>&1; echo pytest_exit=$? >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke_exit=$? >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
DDPMA_KERNEL=P timeout 600 python bench.py --no-cpu --no-e2e > $O/bench_c3_P.json 2> $O/bench_c3_P.err
timeout 600 python bench.py --profile stable --no-cpu --no-e2e > $O/bench_c3_stable.json 2> $O/bench_c3_stable.err
timeout 900 python bench.py --config C5 --no-cpu --no-e2e --steps 2 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --config C4 --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --config C2 --profile stable --until-tol 1e-6 > $O/ttc_c2_stable.json 2> $O/ttc_c2_stable.err
timeout 600 python bench.py --config C1 --until-tol 1e-6 > $O/ttc_c1_default.json 2> $O/ttc_c1_default.err
timeout 300 python bench.py --impl reference --steps 1 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 300 python tools/profile_window.py C3 2 > $O/plainD.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv \
  python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 > $O/ncu_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_windowD -s 2 -c 1 \
  -o $O/r2_c3_windowD python tools/profile_window.py C3 2 > $O/ncuD.log 2>&1
echo done
