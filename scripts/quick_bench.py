import torch, time, sys
sys.path.insert(0, '.')
import paper_2603_01960_b200 as ta
for (B,H,S,D,dt) in [(1,8,512,64,torch.float16),(4,16,4096,64,torch.bfloat16),(8,32,4096,128,torch.bfloat16),(1,16,16384,128,torch.bfloat16),(8,8,32768,128,torch.bfloat16)]:
    q,k,v = (torch.randn(B,H,S,D,device='cuda',dtype=dt) for _ in range(3))
    for _ in range(3): ta.sdpa(q,k,v)
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    n=10
    e0.record()
    for _ in range(n): ta.sdpa(q,k,v)
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/n
    fl=4*B*H*S*S*D
    ref = torch.nn.functional.scaled_dot_product_attention(q,k,v)
    o = ta.sdpa(q,k,v)
    err=(o.float()-ref.float()).abs().max().item()
    e0.record()
    for _ in range(n): torch.nn.functional.scaled_dot_product_attention(q,k,v)
    e1.record(); torch.cuda.synchronize()
    ms2=e0.elapsed_time(e1)/n
    print(f"B{B} H{H} S{S} D{D} {dt}: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOP/s | torch sdpa {ms2:.3f} ms {fl/ms2/1e9:.1f} TFLOP/s | maxdiff {err:.2e}", flush=True)
