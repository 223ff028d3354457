"""Per-call cost of a small launch (BASELINE cfg1: B1 H8 S512 D64 f16):
back-to-back calls (host path included) vs the same calls replayed from a
CUDA graph (device time only), and the pure Python/ctypes wrapper cost.
usage: python scripts/host_overhead.py [B H S D]"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2603_01960_b200 as ta

B, H, S, D = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (1, 8, 512, 64)
q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=torch.float16) for _ in range(3))
o = torch.empty_like(q)
n = 200
for _ in range(20):
    ta.sdpa(q, k, v, out=o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    ta.sdpa(q, k, v, out=o)
e1.record()
torch.cuda.synchronize()
print(f"back-to-back: {e0.elapsed_time(e1) / n * 1e3:.1f} us/call (events)")
t = time.perf_counter()
for _ in range(n):
    ta.sdpa(q, k, v, out=o)
torch.cuda.synchronize()
print(f"host wall: {(time.perf_counter() - t) / n * 1e6:.1f} us/call")
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n):
            ta.sdpa(q, k, v, out=o)
torch.cuda.synchronize()
g.replay()
torch.cuda.synchronize()
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
print(f"graph replay: {e0.elapsed_time(e1) / n * 1e3:.1f} us/call (device time + graph launch spacing)")
for _ in range(3):
    torch.nn.functional.scaled_dot_product_attention(q, k, v)
torch.cuda.synchronize()
e0.record()
for _ in range(n):
    torch.nn.functional.scaled_dot_product_attention(q, k, v)
e1.record()
torch.cuda.synchronize()
print(f"torch sdpa back-to-back: {e0.elapsed_time(e1) / n * 1e3:.1f} us/call")

# where the host time goes (wall clock per call, GPU queue kept short)
import ctypes, timeit
def per_call(fn, n=2000):
    fn()
    t = timeit.timeit(fn, number=n) / n
    torch.cuda.synchronize()
    return t * 1e6
L = ta.lib()
shape = ta._Shape(B, H, S, D)
sched = ta.TileSchedule()._c()
st = ta._Stats()
sp = torch.cuda.current_stream().cuda_stream
qp, kp, vp, op = q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr()
raw = lambda: L.ta_sdpa_fwd(qp, kp, vp, op, None, shape, ta.F16, ta.MASK_NONE, None, 0, 0.0, sched,
                            sp, ctypes.byref(st))
print(f"raw C-ABI call: {per_call(raw):.1f} us")
print(f"ta.sdpa: {per_call(lambda: ta.sdpa(q, k, v, out=o)):.1f} us")
print(f"torch.cuda.current_stream: {per_call(lambda: torch.cuda.current_stream(q.device).cuda_stream):.1f} us")
def dev_ctx():
    with torch.cuda.device(q.device):
        pass
print(f"with torch.cuda.device: {per_call(dev_ctx):.1f} us")
print(f"3x data_ptr + contiguous: {per_call(lambda: (q.contiguous().data_ptr(), k.contiguous().data_ptr(), v.contiguous().data_ptr())):.1f} us")
