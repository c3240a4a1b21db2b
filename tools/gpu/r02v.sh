python - <<'PY'
import time, sys
sys.path.insert(0, '.')
import bench, torch
t0=time.time()
with bench.ClockSampler(0) as c:
    time.sleep(0.2)
print("sleep 0.2s:", len(c.rows), c.summary(), time.time()-t0)
import pynvml
pynvml.nvmlInit(); h=pynvml.nvmlDeviceGetHandleByIndex(0)
t=time.time()
for _ in range(20): pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
print("clockinfo us", (time.time()-t)/20*1e6)
t=time.time()
for _ in range(20): pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
print("reasons us", (time.time()-t)/20*1e6)
x=torch.randn(8192,8192,device='cuda',dtype=torch.bfloat16)
torch.cuda.synchronize()
with bench.ClockSampler(0) as c:
    for _ in range(50): y=x@x
    torch.cuda.synchronize()
print("gemm loop:", len(c.rows), c.summary())
PY
