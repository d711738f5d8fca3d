"""How much does in-process NVML sampling perturb the timed frame loop?  (per-call latency and frame-time impact)"""
import os, sys, time, threading
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, pynvml as n
from paper_2206_10885_b200 import grid, surface
from bench import orbit_view
W, H = 1920, 1080
fs = surface.FieldSurface(grid.field_init(grid.GridConfig(resolution=16), seed=0), device=0)
st = surface.RenderSettings()
dev = torch.device("cuda", 0)
bufs = (torch.empty((H, W, 3), dtype=torch.float32, device=dev), torch.empty((H, W), dtype=torch.float32, device=dev),
        torch.empty((H, W, 3), dtype=torch.float32, device=dev), torch.empty((H, W), dtype=torch.uint8, device=dev))
def loop(k):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for s in range(k):
        surface.render_rows(fs, orbit_view(s, W, H), st, (1.0, 1.0, 1.0), 1, 0, H, out=bufs, device_out=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / k
n.nvmlInit(); h = n.nvmlDeviceGetHandleByIndex(0)
calls = {"clock_sm": lambda: n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM), "max_clock": lambda: n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM),
         "reasons": lambda: n.nvmlDeviceGetCurrentClocksEventReasons(h), "power": lambda: n.nvmlDeviceGetPowerUsage(h)}
print("warm", loop(5))
print("no sampler: %.2f ms/frame" % loop(20))
for name, fn in calls.items():
    t0 = time.perf_counter(); [fn() for _ in range(5)]; idle = (time.perf_counter() - t0) / 5 * 1e3
    stop = threading.Event(); lat = []
    def run():
        while not stop.is_set():
            t = time.perf_counter(); fn(); lat.append((time.perf_counter() - t) * 1e3); stop.wait(0.1)
    th = threading.Thread(target=run, daemon=True); th.start()
    ms = loop(20); stop.set(); th.join()
    print("%-10s idle latency %.2f ms; under load %.2f ms (n=%d); frame %.2f ms" % (name, idle, sum(lat) / max(len(lat), 1), len(lat), ms))
print("no sampler: %.2f ms/frame" % loop(20))
