"""Pinned host <-> device copy times (CUDA events, median of 30) for the e2e copy floor:
H2D / D2H of 0.7-2.7 MB alone, and one concurrent 1.7 MB H2D + 1.7 MB D2H pair on two streams.
    python scripts/pcie_probe.py"""
import torch, time
torch.cuda.init()
s = torch.cuda.Stream(); s2 = torch.cuda.Stream()
for mb in (0.7, 1.0, 1.7, 2.7):
    n = int(mb * 2**20 / 4)
    h = torch.empty(n).pin_memory(); d = torch.empty(n, device='cuda')
    for direction in ("h2d", "d2h"):
        ts = []
        for i in range(30):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                if direction == "h2d": d.copy_(h, non_blocking=True)
                else: h.copy_(d, non_blocking=True)
                e1.record(s)
            s.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(f"{direction} {mb} MB: {ts[len(ts)//2]:.1f} us  {n*4/ts[len(ts)//2]/1e3:.1f} GB/s")
# bidirectional
n = int(1.7 * 2**20 / 4)
h1 = torch.empty(n).pin_memory(); d1 = torch.empty(n, device='cuda'); h2 = torch.empty(n).pin_memory(); d2 = torch.empty(n, device='cuda')
ts=[]
for i in range(30):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    s2.wait_event(e0)
    with torch.cuda.stream(s): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    ev = torch.cuda.Event(); ev.record(s2); s.wait_event(ev)
    e1.record(s)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1)*1e3)
ts.sort(); print(f"bidir 1.7+1.7 MB: {ts[15]:.1f} us")
import subprocess
print(subprocess.run("nvidia-smi -q | grep -A3 -i 'Link Width\\|PCIe Generation' | head -20", shell=True, capture_output=True, text=True).stdout)
