# straight-line two-node log-equidistribution (logequi_pair): quotient check, parity, benches
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -Xcompiler -ffp-contract=off -Iinclude tools/div_check.cu -o /tmp/div_check > $O/div_check.log 2>&1 && /tmp/div_check >> $O/div_check.log 2>&1; echo div_exit=$? >> $O/div_check.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 --timeout-method=thread > $O/pytest_x.log 2>&1; echo pytest_exit=$? >> $O/pytest_x.log
timeout 400 python bench.py --no-cpu --steps 3 --warmup 3 > $O/bench_x_c3.json 2> $O/bench_x_c3.err
timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_x_c3_b.json 2> $O/bench_x_c3_b.err
timeout 500 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 --profile stable > $O/bench_x_c3_stable.json 2> $O/bench_x_c3_stable.err
echo done
