"""Sustained device copy bandwidth (torch copy_ of 4 GiB fp64 buffers back to back
for ~4 s, CUDA events), with the SM clock sampled meanwhile -- the HBM figure a
long-running memory-bound kernel can expect under the board's power cap."""
import json, threading, time
import torch
import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
n = 512 * 1024 * 1024  # 4 GiB of fp64
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty_like(a)
a.fill_(1.0)
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
clk = []
stop = threading.Event()
def sample():
    while not stop.is_set():
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        time.sleep(0.01)
th = threading.Thread(target=sample); th.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 0
e0.record()
t = time.time()
while time.time() - t < 4.0:
    for _ in range(10):
        b.copy_(a); a.copy_(b)
    reps += 20
e1.record()
torch.cuda.synchronize()
stop.set(); th.join()
ms = e0.elapsed_time(e1)
gbs = reps * 2 * n * 8 / (ms * 1e-3) / 1e9
clk.sort()
print(json.dumps({"sustained_copy_GBps": gbs, "copies": reps, "seconds": ms / 1e3, "sm_mhz_median": clk[len(clk) // 2]}))
