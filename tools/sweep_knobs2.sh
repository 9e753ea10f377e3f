#!/bin/bash
# Second knob sweep: combinations of the tail settings that beat the default in
# sweep_knobs.sh, each run twice, plus the GPU parity suite under the best one.
set -u
mkdir -p gpurun_out
out=gpurun_out/sweep_knobs2.jsonl
: > "$out"
run() {
  local tag="$1"; shift
  line=$(env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1)
  echo "{\"tag\": \"$tag\", \"line\": $line}" >> "$out"
}
for rep in 1 2; do
  run base DDPMA_CHUNK=8
  run tail2 DDPMA_CHUNK_TAIL=2
  run tail2_n8 DDPMA_CHUNK_TAIL=2 DDPMA_TAIL_N=8
  run tail2_n12 DDPMA_CHUNK_TAIL=2 DDPMA_TAIL_N=12
  run tail4_n8 DDPMA_CHUNK_TAIL=4 DDPMA_TAIL_N=8
done
