import time, pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
for i in range(5):
    t=time.perf_counter(); a=pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM); t1=time.perf_counter()
    b=pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM); t2=time.perf_counter()
    r=pynvml.nvmlDeviceGetCurrentClocksEventReasons(h); t3=time.perf_counter()
    print(f"{(t1-t)*1e3:.3f} {(t2-t1)*1e3:.3f} {(t3-t2)*1e3:.3f} ms")
