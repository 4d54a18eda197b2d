import torch, time
n = 1 << 30
a = torch.empty(n, dtype=torch.uint8, pin_memory=True)
a.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3): d.copy_(a, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): d.copy_(a, non_blocking=True)
torch.cuda.synchronize()
print("pinned H2D GB/s", 5 * n / (time.perf_counter() - t) / 1e9)
b = torch.empty(n, dtype=torch.uint8)
b.fill_(1)
t = time.perf_counter()
for _ in range(2): d.copy_(b)
torch.cuda.synchronize()
print("pageable H2D GB/s", 2 * n / (time.perf_counter() - t) / 1e9)
import subprocess
print(subprocess.run(["nvidia-smi","--query-gpu=pcie.link.gen.current,pcie.link.width.current","--format=csv"],capture_output=True,text=True).stdout)
print(subprocess.run(["nproc"],capture_output=True,text=True).stdout, open("/proc/cpuinfo").read().count("processor"))

# the ecco C-ABI upload from torch-pinned buffers (bench.py's e2e leg)
import numpy as np, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_11727_b200 as ecco
N, R, S, F = 2000, 512, 64, 512
ctx = ecco.Context(backend=ecco.LEARNED, math=ecco.TC_BF16, max_cameras=N, max_jobs=4, max_depth=2)
ctx.set_cameras(np.zeros((N, 2)), np.full(N, 8.192e6))
fr = torch.empty((N, R, F), dtype=torch.int16, pin_memory=True)
lb = torch.empty((N, R), dtype=torch.int32, pin_memory=True)
ev = torch.empty((N, S, F), dtype=torch.int16, pin_memory=True)
el = torch.empty((N, S), dtype=torch.int32, pin_memory=True)
print("is_pinned", fr.is_pinned())
for _ in range(2):
    ctx.upload_frames_host_ptr(N, fr.data_ptr(), lb.data_ptr(), ev.data_ptr(), el.data_ptr())
t = time.perf_counter()
for _ in range(3):
    ctx.upload_frames_host_ptr(N, fr.data_ptr(), lb.data_ptr(), ev.data_ptr(), el.data_ptr())
dt = (time.perf_counter() - t) / 3
by = fr.numel() * 2 + lb.numel() * 4 + ev.numel() * 2 + el.numel() * 4
print("ecco_upload_frames GB/s", by / dt / 1e9)
