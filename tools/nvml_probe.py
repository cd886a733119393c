import time, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for name, fn in [("sm clock", lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                 ("max sm", lambda: pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)),
                 ("reasons", lambda: pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)),
                 ("power", lambda: pynvml.nvmlDeviceGetPowerUsage(h))]:
    ts = []
    for _ in range(5):
        t = time.perf_counter(); fn(); ts.append((time.perf_counter() - t) * 1e3)
    print(name, [round(x, 3) for x in ts])
