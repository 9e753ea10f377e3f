# 3D: ncu --set full of one C4 window (k_windowP<3>), C4/C5 benches at reduced window length; C3 timeline + stable profile + launch list.
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
timeout 400 python bench.py --config C5 --dtau 1e-5 --no-cpu --no-e2e --steps 2 --warmup 3 > $O/bench_c5_dtau1e-5.json 2> $O/bench_c5_dtau1e-5.err
timeout 300 python bench.py --config C4 --dtau 1e-4 --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_c4_dtau1e-4.json 2> $O/bench_c4_dtau1e-4.err
timeout 300 python bench.py --profile stable --no-cpu --no-e2e > $O/bench_c3_stable.json 2> $O/bench_c3_stable.err
DDPMA_TIMELINE=1 timeout 300 python tools/profile_window.py C3 5 > $O/tl_P.log 2>&1
timeout 300 python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 > $O/plain_launches.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r2_launches_c3.csv \
  python bench.py --no-cpu --no-e2e --steps 2 --warmup 3 > $O/ncu_launches.log 2>&1
timeout 300 python tools/profile_window.py C5 1 1e-5 > $O/plain3.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_windowP -s 1 -c 1 \
  -o $O/r2_c5_windowP3 python tools/profile_window.py C5 1 1e-5 > $O/ncu3.log 2>&1
echo done
