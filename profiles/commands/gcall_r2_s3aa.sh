# bulk chunk size re-check on the final kernels (per-subdomain rule on)
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
for c in 8 6 7 5 8; do
DDPMA_CHUNK=$c timeout 200 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 > $O/bench_aa_c$c.json 2> $O/bench_aa_c$c.err
python -c "
import json
d=json.load(open('$O/bench_aa_c$c.json')); print('chunk $c', '%.4g'%d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])" >> $O/bench_aa.log 2>&1
done
echo done
