# where do the sporadic form_stage stalls land (PIPECUT_B200_SLOW_TRACE: CUDA calls > 1 ms)
PIPECUT_B200_SLOW_TRACE=1 timeout 900 python tools/lat_probe.py C1 C2 C3 C2 C3 > gpurun_out/r2bt.log 2>&1
