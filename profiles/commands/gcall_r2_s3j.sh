# 3D consumed-mbarrier pipeline: parity + C4/C5 benches (with / without the combined-Y pass); scaling projection;
# alternating sweep wavefront vs serial; compute-sanitizer racecheck
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
V=$PWD/paper_2006_14602_b200/variants
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread > $O/pytest_j.log 2>&1; echo pytest_exit=$? >> $O/pytest_j.log
timeout 300 python bench.py --config C4 --dtau 1e-4 --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_j_c4.json 2> $O/bench_j_c4.err
timeout 400 python bench.py --config C5 --dtau 2e-6 --no-cpu --no-e2e --steps 2 --warmup 3 > $O/bench_j_c5.json 2> $O/bench_j_c5.err
DDPMA_LIB=$V/libddpma_nocomb.so timeout 300 python bench.py --config C4 --dtau 1e-4 --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_j_c4_nocomb.json 2> $O/bench_j_c4_nocomb.err
DDPMA_LIB=$V/libddpma_nocomb.so timeout 400 python bench.py --config C5 --dtau 2e-6 --no-cpu --no-e2e --steps 2 --warmup 3 > $O/bench_j_c5_nocomb.json 2> $O/bench_j_c5_nocomb.err
timeout 300 python tools/project_scaling.py C3 6 > $O/project_c3.json 2> $O/project_c3.err
timeout 400 python tools/project_scaling.py C5 4 --dtau 2e-6 > $O/project_c5.json 2> $O/project_c5.err
timeout 400 python bench.py --transmission alternating --no-cpu --no-e2e --steps 2 --warmup 3 > $O/bench_j_c3_alt_wave.json 2> $O/bench_j_c3_alt_wave.err
DDPMA_ALT_SERIAL=1 timeout 600 python bench.py --transmission alternating --no-cpu --no-e2e --steps 2 --warmup 3 > $O/bench_j_c3_alt_serial.json 2> $O/bench_j_c3_alt_serial.err
timeout 300 python bench.py --config C2 --until-tol 1e-6 --max-windows 400 > $O/ttc_c2_default.json 2> $O/ttc_c2_default.err
echo done
