timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_gpu.log
for cfg in "W1:DDPMA_WS=1 DDPMA_CHUNK_TAIL=1" "W2:DDPMA_WS=1 DDPMA_CHUNK_TAIL=2" "W4:DDPMA_WS=1 DDPMA_CHUNK_TAIL=4" "P1:DDPMA_WS=0 DDPMA_CHUNK_TAIL=1" "P4:DDPMA_WS=0 DDPMA_CHUNK_TAIL=4"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench_v7_$name.json 2> gpurun_out/bench_v7_$name.err
done
