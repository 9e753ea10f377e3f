# stable-profile C3: per-window times, current build vs the pre-face-path build (bisecting a timeout)
mkdir -p gpurun_out
O=gpurun_out
export PYTHONUNBUFFERED=1
V=$PWD/paper_2006_14602_b200/variants
DDPMA_LIB=$V/libddpma_old.so timeout 150 python tools/window_times.py C3 8 stable > $O/wt_c3_stable_old.log 2>&1
timeout 150 python tools/window_times.py C3 8 stable > $O/wt_c3_stable_cur.log 2>&1
timeout 100 python tools/window_times.py C2 40 stable > $O/wt_c2_stable_cur.log 2>&1
echo done
