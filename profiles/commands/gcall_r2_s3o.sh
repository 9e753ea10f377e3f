# latency breakdown of the top-priority subdomain's actions (DDPMA_PROBE), bulk and tail
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
DDPMA_PROBE=1 timeout 300 python tools/profile_window.py C3 3 > $O/probe_c3.log 2>&1
DDPMA_PROBE=1 DDPMA_SERIAL_ADVANCE=1 timeout 300 python tools/profile_window.py C2 1 > $O/probe_c2_serial.log 2>&1
echo done
