mkdir -p gpurun_out
DDPMA_TIMELINE=1 timeout 300 python tools/profile_window.py C3 3 > gpurun_out/tl_D.log 2>&1
DDPMA_KERNEL=P DDPMA_TIMELINE=1 timeout 300 python tools/profile_window.py C3 3 > gpurun_out/tl_P.log 2>&1
timeout 300 python tools/profile_window.py C3 2 > gpurun_out/plainD.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_windowD -s 2 -c 1 \
  -o gpurun_out/r2_c3_windowD python tools/profile_window.py C3 2 > gpurun_out/ncuD.log 2>&1
echo done
