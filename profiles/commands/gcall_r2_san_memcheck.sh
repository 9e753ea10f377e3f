# compute-sanitizer --tool memcheck on C1 + T3 solves through the persistent window kernels
mkdir -p gpurun_out
timeout 300 python tools/sanitize_case.py 3 2 > gpurun_out/san_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_case.py 3 2 > gpurun_out/san_memcheck.log 2>&1
echo san_exit=$? >> gpurun_out/san_memcheck.log
echo done
