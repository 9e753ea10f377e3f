mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sampled.py tests/test_arc.py tests/test_smooth.py -m gpu -q -s > gpurun_out/pytest_new.log 2>&1; echo exit=$? >> gpurun_out/pytest_new.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_exit=$? >> gpurun_out/smoke.log
timeout 900 python bench.py --config C5 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 600 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
