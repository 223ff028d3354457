import sys, time, torch
sys.path.insert(0, ".")
import paper_2603_01960_b200 as ta
B, H, S, D = 8, 64, 32768, 128
hq, hk, hv = (torch.randn(B, H, S, D, dtype=torch.bfloat16).pin_memory() for _ in range(3))
ho = torch.empty_like(hq).pin_memory()
ptrs = (hq.data_ptr(), hk.data_ptr(), hv.data_ptr(), ho.data_ptr())
st = torch.cuda.current_stream()
ta.sdpa_fwd_host(*ptrs, 0, (B, H, S, D), ta.BF16, stream=st.cuda_stream)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    ta.sdpa_fwd_host(*ptrs, 0, (B, H, S, D), ta.BF16, stream=st.cuda_stream)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 3
print(f"e2e {dt*1e3:.1f} ms  {4*B*H*S*S*D/dt/1e12:.1f} TF/s")
