"""Size-independent properties at the BASELINE sequence lengths, and the
reference's own tiled-vs-oracle grid mirrored on the GPU.

* test_tiled.cpp:273-291 mirrored: S in {32, 130} (ragged), D=48, B1 H2,
  f16/bf16 x {none, causal, padding} x both layouts, schedule (64,64,2).
* test_reference.cpp:148-163 (convex hull), :130-146 (permutation) and
  :84-89 (causal row 0 = v0) as properties of the kernel at S = 16K / 32K,
  where a full oracle is too slow: O lies in the per-column hull of V;
  permuting query rows permutes O bitwise (rows are independent: one TMEM
  lane each); causal row 0 and a padded batch with one admitted key return
  that key's V exactly; a padded batch with none returns zeros / -inf.
"""
import math

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

TOL = {O.F16: 5e-3, O.BF16: 2e-2}


def _t(dt):
    import torch
    return {O.F16: torch.float16, O.BF16: torch.bfloat16}[dt]


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("mask", [O.MASK_NONE, O.MASK_CAUSAL, O.MASK_PADDING])
@pytest.mark.parametrize("dt", [O.F16, O.BF16])
@pytest.mark.parametrize("S", [32, 130])
def test_reference_tiled_grid_mirror(ta, cuda_device, S, dt, mask, layout):
    # test_tiled.cpp:273-291: B1 H2 D48, schedule (64, 64, 2), both layouts
    import torch
    B, H, D = 1, 2, 48
    q, k, v = O.make_input((B, H, S, D), dt, 42)
    vl = [S // 2 + 1] if mask == O.MASK_PADDING else None
    qd, kd, vd = (torch.from_numpy(x).to(_t(dt)).cuda() for x in (q, k, v))
    st = ta.KernelStats()
    o, lse = ta.sdpa(qd, kd, vd, causal=mask == O.MASK_CAUSAL, valid_len=vl, return_lse=True,
                     schedule=ta.TileSchedule(64, 64, 2, layout), stats=st)
    torch.cuda.synchronize()
    r = O.sdpa_reference(q, k, v, mask_kind=mask, valid_len=vl)
    assert np.abs(o.double().cpu().numpy() - r["o"]).max() <= TOL[dt]
    assert np.abs(lse.double().cpu().numpy() - r["lse"]).max() <= 1e-3
    assert st.block_m == 128 and st.block_n == 128  # D=48 runs the 64-column kernel


@pytest.mark.parametrize("shape,dt", [((1, 8, 32768, 128), O.BF16), ((1, 8, 16384, 64), O.F16)])
def test_convex_hull_at_full_length(ta, cuda_device, shape, dt):
    # test_reference.cpp:148-163: each O element lies between the column's
    # min and max over the values (weights are a convex combination)
    import torch
    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.randn(shape, device="cuda", generator=g).to(_t(dt)) for _ in range(3))
    o = ta.sdpa(q, k, v).float()
    vmin = v.float().amin(dim=2, keepdim=True)
    vmax = v.float().amax(dim=2, keepdim=True)
    slack = (vmax - vmin).abs() * 2 ** -7 + 1e-6  # output rounding to the 16-bit grid
    assert bool((o >= vmin - slack).all()) and bool((o <= vmax + slack).all())


def test_query_permutation_is_bitwise_at_32k(ta, cuda_device):
    # rows are independent (one TMEM lane, one thread each): permuting the
    # query rows permutes O and LSE bitwise, across CTAs and tile positions
    import torch
    B, H, S, D = 1, 4, 32768, 128
    g = torch.Generator(device="cuda").manual_seed(11)
    q, k, v = (torch.randn(B, H, S, D, device="cuda", generator=g).bfloat16() for _ in range(3))
    perm = torch.randperm(S, device="cuda", generator=g)
    o1, l1 = ta.sdpa(q, k, v, return_lse=True)
    o2, l2 = ta.sdpa(q[:, :, perm].contiguous(), k, v, return_lse=True)
    torch.cuda.synchronize()
    assert torch.equal(o1[:, :, perm], o2)
    assert torch.equal(l1[:, :, perm], l2)


def test_causal_row0_and_sampled_rows_at_32k(ta, cuda_device):
    # test_reference.cpp:84-89 at the bench length: causal row 0 attends to
    # key 0 only -> O = v0 exactly; sampled later rows vs float64
    import torch
    B, H, S, D = 1, 2, 32768, 128
    g = torch.Generator(device="cuda").manual_seed(13)
    q, k, v = (torch.randn(B, H, S, D, device="cuda", generator=g).bfloat16() for _ in range(3))
    o, lse = ta.sdpa(q, k, v, causal=True, return_lse=True)
    torch.cuda.synchronize()
    assert torch.equal(o[:, :, 0], v[:, :, 0])
    sc = 1.0 / math.sqrt(D)
    for h in range(H):
        kh, vh = k[0, h].double(), v[0, h].double()
        for i in (1, 127, 128, 255, 4097, 20000, S - 1):
            s = (q[0, h, i].double() @ kh[: i + 1].T) * sc
            p = torch.softmax(s, 0)
            want = p @ vh[: i + 1]
            assert (o[0, h, i].double() - want).abs().max().item() <= 2e-2, (h, i)
            assert abs(lse[0, h, i].item() - torch.logsumexp(s, 0).item()) <= 1e-3, (h, i)


def test_padding_extremes_at_16k(ta, cuda_device):
    # valid_len = S, 10000, 1 and 0 in one launch: the single admitted key
    # gives O = v0 exactly and LSE = its scaled score; no admitted key gives
    # zeros and -inf (finalize, tiled.hpp:231-233); a ragged length matches
    # float64 on sampled rows
    import torch
    B, H, S, D = 4, 2, 16384, 64
    g = torch.Generator(device="cuda").manual_seed(17)
    q, k, v = (torch.randn(B, H, S, D, device="cuda", generator=g).bfloat16() for _ in range(3))
    vl = [S, 10000, 1, 0]
    o, lse = ta.sdpa(q, k, v, valid_len=vl, return_lse=True)
    torch.cuda.synchronize()
    sc = 1.0 / math.sqrt(D)
    assert torch.equal(o[2], v[2, :, :1].expand(H, S, D))
    s00 = (q[2].double() @ k[2, :, 0].double().unsqueeze(-1)).squeeze(-1) * sc
    assert (lse[2].double() - s00).abs().max().item() <= 1e-4
    assert bool((o[3] == 0).all()) and bool(torch.isneginf(lse[3]).all())
    for b in (0, 1):
        n = vl[b]
        for h in range(H):
            kh, vh = k[b, h, :n].double(), v[b, h, :n].double()
            for i in (0, 129, 9999, 12000, S - 1):
                s = (q[b, h, i].double() @ kh.T) * sc
                want = torch.softmax(s, 0) @ vh
                assert (o[b, h, i].double() - want).abs().max().item() <= 2e-2, (b, h, i)
                assert abs(lse[b, h, i].item() - torch.logsumexp(s, 0).item()) <= 1e-3


def test_nan_propagates_like_the_reference(ta, cuda_device):
    # a NaN in one query row poisons that row only (its scores are NaN, the
    # reference's exp / sum propagate it); a NaN key poisons every row whose
    # mask admits it -- and with causal masking only the rows at or after it
    import torch
    B, H, S, D = 1, 2, 1000, 64
    g = torch.Generator(device="cuda").manual_seed(19)
    q, k, v = (torch.randn(B, H, S, D, device="cuda", generator=g).half() for _ in range(3))
    qn = q.clone()
    qn[0, 0, 123, 5] = float("nan")
    o, lse = ta.sdpa(qn, k, v, return_lse=True)
    torch.cuda.synchronize()
    bad = torch.zeros(S, dtype=torch.bool, device="cuda")
    bad[123] = True
    assert bool(torch.isnan(o[0, 0, 123]).all()) and bool(torch.isnan(lse[0, 0, 123]))
    assert bool(torch.isfinite(o[0, 0, ~bad]).all()) and bool(torch.isfinite(o[0, 1]).all())
    ref = ta.sdpa(q, k, v)
    assert torch.equal(o[0, 0, ~bad], ref[0, 0, ~bad])  # other rows untouched, bit for bit
    kn = k.clone()
    kn[0, 1, 700, 0] = float("nan")
    o2 = ta.sdpa(q, kn, v, causal=True)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(o2[0, 1, :700]).all())
    assert bool(torch.isnan(o2[0, 1, 700:]).any(dim=-1).all())


@pytest.mark.parametrize("D,t_n", [(64, 128), (128, 128), (128, 64), (160, 128), (256, 128)])
def test_padding_ignores_nan_beyond_valid_len(ta, cuda_device, D, t_n):
    # keys >= valid_len have weight 0, and the reference skips zero weights
    # (online_update, tiled.hpp:215-216): NaN / inf in the padded K and V
    # rows must not reach O or LSE -- the result equals the clean inputs', bit
    # for bit, on every kernel (rotation, two-tile, 64-key, wide)
    import torch
    B, H, S = 3, 2, 700
    g = torch.Generator(device="cuda").manual_seed(23 + D)
    q, k, v = (torch.randn(B, H, S, D, device="cuda", generator=g).bfloat16() for _ in range(3))
    vl = [300, 129, 700]
    sched = ta.TileSchedule(64, t_n, 2)
    o1, l1 = ta.sdpa(q, k, v, valid_len=vl, return_lse=True, schedule=sched)
    kg, vg = k.clone(), v.clone()
    for b, n in enumerate(vl):
        kg[b, :, n:] = float("nan")
        vg[b, :, n:] = float("inf")
        vg[b, :, n + 1:n + 3] = float("nan")
    o2, l2 = ta.sdpa(q, kg, vg, valid_len=vl, return_lse=True, schedule=sched)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    assert bool(torch.isfinite(o2).all())


def test_very_long_sequence_sampled_rows(ta, cuda_device):
    # S = 2^17 (1024 K/V tiles per row, 4x the bench length): sampled rows of
    # every 256-row CTA class against float64
    import torch
    B, H, S, D = 1, 1, 131072, 128
    g = torch.Generator(device="cuda").manual_seed(29)
    q, k, v = (torch.randn(B, H, S, D, device="cuda", generator=g).bfloat16() for _ in range(3))
    o, lse = ta.sdpa(q, k, v, return_lse=True)
    torch.cuda.synchronize()
    kd, vd = k[0, 0].double(), v[0, 0].double()
    for i in (0, 1, 255, 256, 65535, 99999, S - 1):
        s = (q[0, 0, i].double() @ kd.T) / math.sqrt(D)
        want = torch.softmax(s, 0) @ vd
        assert (o[0, 0, i].double() - want).abs().max().item() <= 2e-2, i
        assert abs(lse[0, 0, i].item() - torch.logsumexp(s, 0).item()) <= 1e-3, i


@pytest.mark.parametrize("D", [64, 128, 256])
def test_extreme_scale_is_one_hot(ta, cuda_device, D):
    # scale 100: every row's softmax is (numerically) one-hot, the running max
    # jumps on many tiles (stale-max slow path), and exps of the other keys
    # underflow to exact 0 -- O must be the argmax key's V row
    import torch
    B, H, S = 1, 2, 3000
    g = torch.Generator(device="cuda").manual_seed(31 + D)
    q, k, v = (torch.randn(B, H, S, D, device="cuda", generator=g).half() for _ in range(3))
    o, lse = ta.sdpa(q, k, v, scale=100.0, return_lse=True)
    torch.cuda.synchronize()
    s = torch.einsum("bhqd,bhkd->bhqk", q.double(), k.double()) * 100.0
    top2 = s.topk(2, dim=-1).values
    clear = (top2[..., 0] - top2[..., 1]) > 1.0  # rows whose max is unambiguous
    want = torch.softmax(s, -1) @ v.double()
    err = (o.double() - want).abs().amax(-1)
    assert bool((err[clear] <= 5e-3).all()), err[clear].max().item()
    # LSE ~ 6000 here: fp32 carries it to ~5e-7 relative (scores from the fp32
    # tensor-core sums times scale * log2 e in fp32)
    want_lse = torch.logsumexp(s, -1)
    assert bool(((lse.double() - want_lse).abs() <= 2e-3 + 2e-6 * want_lse.abs()).all())


@pytest.mark.parametrize("D", [64, 128])
def test_nan_in_any_key_column(ta, cuda_device, D):
    # a NaN key at every column position of a 128-key tile (some land on the
    # FMA-pipe exp emulation at D=64): every query row admits it, so every
    # row's O and LSE are NaN, as the reference's arithmetic gives
    import torch
    B, H, S = 1, 1, 256
    for col in range(0, 128, 3):
        g = torch.Generator(device="cuda").manual_seed(37 + col)
        q, k, v = (torch.randn(B, H, S, D, device="cuda", generator=g).half() for _ in range(3))
        k[0, 0, 128 + col, 0] = float("nan")
        o, lse = ta.sdpa(q, k, v, return_lse=True)
        torch.cuda.synchronize()
        assert bool(torch.isnan(lse).all()), col
        assert bool(torch.isnan(o).any(dim=-1).all()), col
