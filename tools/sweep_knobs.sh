#!/bin/bash
# Runtime-knob sweep of the C3 window kernel (no rebuild): chunk sizes and tail
# threshold of the persistent window scheduler (plan.cu), single-role vs
# warp-specialised 2D kernel. One bench line per setting into gpurun_out/.
set -u
mkdir -p gpurun_out
out=gpurun_out/sweep_knobs.jsonl
: > "$out"
run() {
  local tag="$1"; shift
  line=$(env "$@" timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1)
  echo "{\"tag\": \"$tag\", \"line\": $line}" >> "$out"
}
run base DDPMA_CHUNK=8
run chunk4 DDPMA_CHUNK=4
run chunk16 DDPMA_CHUNK=16
run tail2 DDPMA_CHUNK_TAIL=2
run tailn8 DDPMA_TAIL_N=8
run tailn32 DDPMA_TAIL_N=32
run ws DDPMA_WS=1
