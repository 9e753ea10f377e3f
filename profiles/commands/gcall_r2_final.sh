# Round-2 evidence run on a fresh B200: GPU tests, smoke, headline bench (with e2e + cpu baseline), reference arm,
# 3D / stable / time-to-converged lines, ncu launch list and --set full captures of the 2D and 3D window kernels.
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/final_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rA --durations=10 --timeout 300 --timeout-method=thread > $O/final_pytest_gpu.log 2>&1; echo pytest_exit=$? >> $O/final_pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.log 2>&1; echo smoke_exit=$? >> $O/final_smoke.log
timeout 600 python bench.py > $O/final_bench_c3.json 2> $O/final_bench_c3.err
timeout 300 python bench.py --impl reference --steps 1 --warmup 1 > $O/final_bench_ref.json 2> $O/final_bench_ref.err
timeout 600 python bench.py --config C5 --dtau 2e-6 --no-e2e --steps 2 --warmup 3 > $O/final_bench_c5.json 2> $O/final_bench_c5.err
timeout 400 python bench.py --config C4 --dtau 1e-4 --steps 3 --warmup 3 > $O/final_bench_c4.json 2> $O/final_bench_c4.err
timeout 500 python bench.py --profile stable --no-cpu --no-e2e > $O/final_bench_c3_stable.json 2> $O/final_bench_c3_stable.err
timeout 200 python bench.py --config C1 --until-tol 1e-6 > $O/final_ttc_c1_default.json 2> $O/final_ttc_c1_default.err
timeout 300 python bench.py --config C1 --profile stable --until-tol 1e-6 > $O/final_ttc_c1_stable.json 2> $O/final_ttc_c1_stable.err
timeout 300 python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 > $O/final_plain_launches.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/final_launches_c3.csv \
  python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 > $O/final_ncu_launches.log 2>&1
timeout 300 python tools/profile_window.py C3 2 > $O/final_plain2.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_windowP -s 2 -c 1 \
  -o $O/final_c3_windowP python tools/profile_window.py C3 2 > $O/final_ncu2.log 2>&1
timeout 300 python tools/profile_window.py C5 1 2e-6 > $O/final_plain3.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_windowP -s 1 -c 1 \
  -o $O/final_c5_windowP3 python tools/profile_window.py C5 1 2e-6 > $O/final_ncu3.log 2>&1
echo done
