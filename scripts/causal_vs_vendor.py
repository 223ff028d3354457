import sys, torch
sys.path.insert(0, ".")
import paper_2603_01960_b200 as ta
for (B, H, S, D) in [(8, 32, 4096, 128), (1, 16, 16384, 128), (4, 16, 4096, 64), (8, 64, 32768, 128)]:
    q, k, v = (torch.randn(B, H, S, D, device="cuda", dtype=torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    for causal in (False, True):
        for _ in range(2): ta.sdpa(q, k, v, out=o, causal=causal)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 3 if S >= 32768 else 10
        e0.record()
        for _ in range(n): ta.sdpa(q, k, v, out=o, causal=causal)
        e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / n
        for _ in range(2): torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal)
        e0.record()
        for _ in range(n): torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal)
        e1.record(); torch.cuda.synchronize(); ms2 = e0.elapsed_time(e1) / n
        fl = 4 * B * H * S * S * D / (2 if causal else 1)
        print(f"B{B} H{H} S{S} D{D} causal={causal}: ours {fl/ms/1e9:7.1f} torch {fl/ms2/1e9:7.1f} TF/s (effective)")
