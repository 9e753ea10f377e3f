# D-kernel fix probe (nfold), envelope-based prefix tests, 3D stable-profile benches, time-to-converged.
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
DDPMA_KERNEL=D timeout 90 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_D.log 2>&1; rc=$?; echo smoke_exit=$rc >> $O/smoke_D.log
if [ $rc -eq 0 ]; then
DDPMA_KERNEL=D timeout 600 python -m pytest tests/test_gpu_parity.py -q -rA --timeout 120 --timeout-method=thread -k "c1_prefix or baseline_window or deterministic or one_by_one or c1_default_prefix or rerun or uniform or c1_reference_defaults" > $O/pytest_D.log 2>&1; echo pytest_exit=$? >> $O/pytest_D.log
DDPMA_KERNEL=D timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_D_b4.json 2> $O/bench_D_b4.err
fi
DDPMA_KERNEL=P timeout 300 python -m pytest tests/test_gpu_parity.py -q -rA --timeout 120 --timeout-method=thread -k "c1_variants or c1_prefix" > $O/pytest_P_prefix.log 2>&1; echo pytest_exit=$? >> $O/pytest_P_prefix.log
timeout 400 python bench.py --config C5 --profile stable --no-cpu --no-e2e --steps 2 --warmup 3 > $O/bench_c5_stable.json 2> $O/bench_c5_stable.err
timeout 300 python bench.py --config C4 --profile stable --no-cpu --no-e2e --steps 5 --warmup 3 > $O/bench_c4_stable.json 2> $O/bench_c4_stable.err
timeout 300 python bench.py --config C2 --profile stable --until-tol 1e-6 > $O/ttc_c2_stable.json 2> $O/ttc_c2_stable.err
timeout 300 python bench.py --config C1 --until-tol 1e-6 > $O/ttc_c1_default.json 2> $O/ttc_c1_default.err
echo done
