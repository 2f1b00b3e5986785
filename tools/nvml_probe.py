import torch, pynvml
pynvml.nvmlInit()
p = torch.cuda.get_device_properties(0)
print("uuid", getattr(p, "uuid", None))
h = pynvml.nvmlDeviceGetHandleByUUID("GPU-" + str(p.uuid))
print("sm", pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), "max", pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
f = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
print("reasons", hex(f(h)), "power", pynvml.nvmlDeviceGetPowerUsage(h))
print([n for n in dir(pynvml) if "ClocksEventReason" in n or "ClocksThrottleReason" in n][:20])
