import sys, time, ctypes
sys.path.insert(0, '.')
import torch
import paper_2005_01442_b200 as vr
from paper_2005_01442_b200 import _lib
dv = vr.device_phantom("torso", (512, 512, 512))
L = _lib.load(); s = torch.cuda.current_stream(); sp = _lib.ptr_stream(s)
out = torch.zeros(2, dtype=torch.int64, device="cuda"); cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); ev[0].record(s)
    for _ in range(n): fn()
    ev[1].record(s); ev[1].synchronize(); return ev[0].elapsed_time(ev[1]) / n * 1e3
print("count us", t(lambda: L.vr_threshold_count(dv.handle, 550, _lib.ptr(cnt), sp)))
print("measure us", t(lambda: L.vr_threshold_measure(dv.handle, 550, _lib.ptr(out), sp)))
x = torch.empty(1 << 24, dtype=torch.int32, device="cuda")
print("memset-only us", t(lambda: out.zero_()))
print("malloc/free 16MB us", t(lambda: torch.empty(1 << 22, dtype=torch.int32, device="cuda")))
