"""sm_100a memory-bound and attention kernels vs plain PyTorch fp32 references."""
import ctypes as C

import pytest
import torch
import torch.nn.functional as F

from paper_2102_03161_b200 import ops

pytestmark = pytest.mark.gpu


def _s():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _rel(a, b):
    return ((a.float() - b.float()).norm() / (b.float().norm() + 1e-12)).item()


@pytest.mark.parametrize("d", [128, 768, 1024])
def test_layernorm_fwd_bwd(cuda, d):
    g = torch.Generator(device=cuda).manual_seed(d)
    R = 3001
    x = (torch.randn(R, d, device=cuda, generator=g) * 2 + 0.5).bfloat16()
    gamma = torch.randn(d, device=cuda, generator=g)
    beta = torch.randn(d, device=cuda, generator=g)
    y = torch.empty_like(x)
    mean = torch.empty(R, device=cuda)
    rstd = torch.empty(R, device=cuda)
    ops.call("eps_layernorm_fwd", x, gamma, beta, y, mean, rstd, R, d, C.c_float(1e-6), _s())
    xf = x.float().requires_grad_()
    gf, bf = gamma.clone().requires_grad_(), beta.clone().requires_grad_()
    ref = F.layer_norm(xf, (d,), gf, bf, eps=1e-6)
    torch.cuda.synchronize()
    assert _rel(y, ref) < 1e-2
    dy = torch.randn(R, d, device=cuda, generator=g).bfloat16()
    dres = torch.randn(R, d, device=cuda, generator=g).bfloat16()
    ref.backward(dy.float())
    dx = torch.empty_like(x)
    dgam = torch.zeros(d, device=cuda)
    dbet = torch.zeros(d, device=cuda)
    cs = torch.zeros(d, device=cuda)
    ops.call("eps_layernorm_bwd", dy, x, gamma, mean, rstd, dres, dx, dgam, dbet, cs, R, d, None,
             _s())
    torch.cuda.synchronize()
    want = xf.grad + dres.float()
    assert _rel(dx, want) < 1e-2
    assert _rel(dgam, gf.grad) < 1e-2
    assert _rel(dbet, bf.grad) < 1e-2
    assert _rel(cs, want.sum(0)) < 1e-2  # fp32 column sums of the produced dx


@pytest.mark.parametrize("d", [768, 1024])
def test_layernorm_fwd_offset_rows(cuda, d):
    """Rows whose mean is large against their spread (offsets up to 300 sigma,
    a constant row, one outlier column): the one-pass (shifted) statistics of
    ln_fwd_wide_kernel must match fp32 LayerNorm; mean / rstd are checked too."""
    g = torch.Generator(device=cuda).manual_seed(7)
    R = 1000
    off = torch.linspace(-300, 300, R, device=cuda).unsqueeze(1)
    x = torch.randn(R, d, device=cuda, generator=g) * 0.5 + off
    x[5] = 3.0                   # zero variance
    x[6, 17] += 1e4              # one outlier column
    x[7, 0] = x[7, 1:].mean() + 50.0  # the shift element itself is the outlier
    x = x.bfloat16()
    gamma = torch.randn(d, device=cuda, generator=g)
    beta = torch.randn(d, device=cuda, generator=g)
    y = torch.empty_like(x)
    mean = torch.empty(R, device=cuda)
    rstd = torch.empty(R, device=cuda)
    ops.call("eps_layernorm_fwd", x, gamma, beta, y, mean, rstd, R, d, C.c_float(1e-6), _s())
    xf = x.float()
    ref = F.layer_norm(xf, (d,), gamma, beta, eps=1e-6)
    torch.cuda.synchronize()
    assert torch.isfinite(y.float()).all()
    assert _rel(y, ref) < 1e-2
    per_row = (y.float() - ref).norm(dim=1) / ref.norm(dim=1).clamp_min(1e-6)
    assert per_row.max().item() < 2e-2
    assert ((mean - xf.mean(1)).abs() / xf.std(1).clamp_min(1e-3)).max().item() < 1e-3
    want_rstd = torch.rsqrt(xf.var(1, unbiased=False) + 1e-6)
    assert ((rstd - want_rstd).abs() / want_rstd).max().item() < 1e-3


def _attn_ref(qkv, B, T, H, dh):
    D = H * dh
    q, k, v = qkv.float().reshape(B, T, 3 * D).split(D, dim=-1)
    q = q.reshape(B, T, H, dh).transpose(1, 2)
    k = k.reshape(B, T, H, dh).transpose(1, 2)
    v = v.reshape(B, T, H, dh).transpose(1, 2)
    s = (q @ k.transpose(-1, -2)) * dh ** -0.5
    o = torch.softmax(s, -1) @ v
    return o.transpose(1, 2).reshape(B * T, D), torch.logsumexp(s, -1)


# (30, 197, 12) and (64, 128, 16) put several heads on every CTA of the
# persistent kernels (their smem / TMEM / table double-buffering); 256, 129
# and 1 are the tile-boundary edges of the fused backward.
@pytest.mark.parametrize("B,T,H,dh", [(3, 197, 12, 64), (5, 65, 4, 32), (2, 128, 16, 64),
                                      (1, 384, 12, 64), (2, 50, 2, 64), (30, 197, 12, 64),
                                      (64, 128, 16, 64), (3, 256, 4, 64), (7, 129, 3, 64),
                                      (5, 1, 2, 64), (1, 255, 1, 64), (300, 197, 1, 64),
                                      (40, 64, 8, 64),
                                      # 256 < T <= 384: (head, key tile) units, several per
                                      # CTA, ragged last key / query tile, dQ slice reduce
                                      (8, 384, 12, 64), (3, 300, 4, 64), (2, 257, 3, 64),
                                      # T <= 128: head pairs per unit; odd head count falls back
                                      (3, 100, 3, 64), (37, 128, 4, 64)])
def test_attention_fwd_bwd(cuda, B, T, H, dh):
    g = torch.Generator(device=cuda).manual_seed(T * H)
    D = H * dh
    qkv = torch.randn(B * T, 3 * D, device=cuda, generator=g).bfloat16()
    out = torch.empty(B * T, D, device=cuda, dtype=torch.bfloat16)
    lse = torch.empty(B, H, T, device=cuda)
    scale = dh ** -0.5
    ops.call("eps_attn_fwd", qkv, out, lse, B, T, H, dh, C.c_float(scale), _s())
    qf = qkv.float().requires_grad_()
    ref, ref_lse = _attn_ref(qf, B, T, H, dh)
    torch.cuda.synchronize()
    assert _rel(out, ref) < 1e-2
    assert (lse - ref_lse).abs().max().item() < 2e-2
    dout = torch.randn(B * T, D, device=cuda, generator=g).bfloat16()
    ref.backward(dout.float())
    dqkv = torch.empty_like(qkv)
    dbias = torch.zeros(3 * D, device=cuda)
    dsum = torch.empty(B * H * T, device=cuda)
    ops.call("eps_attn_bwd_ws", qkv, out, dout, lse, dqkv, dbias, dsum, B, T, H, dh,
             C.c_float(scale), _s())
    torch.cuda.synchronize()
    for part in range(3):
        sl = slice(part * D, (part + 1) * D)
        if T == 1 and part < 2:  # one key: softmax == 1, exact dQ = dK = 0
            assert dqkv[:, sl].float().abs().max().item() < 2e-2 * dout.float().abs().max().item()
            continue
        assert _rel(dqkv[:, sl], qf.grad[:, sl]) < 2e-2, part
    assert _rel(dbias, dqkv.float().sum(0)) < 1e-3
    # precomputed-D entry (D = rowsum(dO * O) per (row, head), [B*T, H]) agrees
    if ops.api().lib.eps_attn_bwd_uses_rowdot(T, dh):
        drow = (dout.float() * out.float()).reshape(B * T, H, dh).sum(-1).contiguous()
        dqkv2 = torch.empty_like(qkv)
        dbias2 = torch.zeros(3 * D, device=cuda)
        ops.call("eps_attn_bwd_rowdot", qkv, out, dout, lse, drow, dqkv2, dbias2, dsum, B, T, H,
                 dh, C.c_float(scale), _s())
        torch.cuda.synchronize()
        assert _rel(dqkv2, dqkv) < 1e-2
        assert _rel(dbias2, dbias) < 1e-2


def test_attention_bwd_paired_heads(cuda, monkeypatch):
    """The paired-head backward (T <= 128, EPS_ATTN_BWD_PAIRS=1; off by default)
    matches the per-head one, in a fresh process so the switch is read."""
    import subprocess
    import sys
    code = (
        "import torch, ctypes as C, sys; sys.path.insert(0, '.');"
        "from paper_2102_03161_b200 import ops;"
        "B, T, H = 6, 100, 4; D = H * 64; g = torch.Generator(device='cuda').manual_seed(3);"
        "qkv = torch.randn(B*T, 3*D, device='cuda', generator=g).bfloat16();"
        "out = torch.empty(B*T, D, device='cuda', dtype=torch.bfloat16);"
        "lse = torch.empty(B, H, T, device='cuda'); s = C.c_void_p(0); sc = C.c_float(0.125);"
        "ops.call('eps_attn_fwd', qkv, out, lse, B, T, H, 64, sc, s);"
        "do = torch.randn(B*T, D, device='cuda', generator=g).bfloat16();"
        "dq = torch.empty_like(qkv); db = torch.zeros(3*D, device='cuda');"
        "ds = torch.empty(B*H*T, device='cuda');"
        "ops.call('eps_attn_bwd_ws', qkv, out, do, lse, dq, db, ds, B, T, H, 64, sc, s);"
        "torch.cuda.synchronize(); torch.save((dq.cpu(), db.cpu()), sys.argv[1])")
    outs = []
    import tempfile, os
    with tempfile.TemporaryDirectory() as d:
        for flag in ("0", "1"):
            f = os.path.join(d, f"r{flag}.pt")
            env = dict(os.environ, EPS_ATTN_BWD_PAIRS=flag)
            r = subprocess.run([sys.executable, "-c", code, f], cwd=os.path.dirname(
                os.path.dirname(os.path.abspath(__file__))), env=env, capture_output=True,
                text=True, timeout=300)
            assert r.returncode == 0, r.stderr[-2000:]
            outs.append(torch.load(f))
    (a, ba), (b, bb) = outs
    assert _rel(b, a) < 1e-2
    assert _rel(bb, ba) < 1e-2


@pytest.mark.parametrize("T,spike", [(197, 40), (197, 196), (128, 100), (256, 255), (384, 100),
                                     (384, 250), (384, 383), (300, 299)])
def test_attention_fwd_score_spike(cuda, T, spike):
    """Keys whose score exceeds every score of the first 32 keys by far more than
    2^32 (in exp2 units): the forward's one-pass softmax must rescale the P
    chunks it already wrote.  Rows get spikes of different sizes, some none."""
    B, H, dh = 2, 3, 64
    D = H * dh
    g = torch.Generator(device=cuda).manual_seed(spike)
    qkv = torch.randn(B * T, 3 * D, device=cuda, generator=g)
    qkv = qkv.reshape(B, T, 3 * D)
    q = qkv[:, :, :D].reshape(B, T, H, dh)
    k = qkv[:, :, D:2 * D].reshape(B, T, H, dh)
    # queries share a direction u per (sample, head); key `spike` is u scaled
    # with the head index, so its score leads by ~46 / 92 / 138 exp2 units
    u = torch.randn(B, 1, H, dh, device=cuda, generator=g)
    q.mul_(0.5).add_(u)
    k[:, spike] = u[:, 0] * (4.0 * (torch.arange(H, device=cuda) + 1)).reshape(1, H, 1)
    q[:, ::3] *= 2.0
    qkv = qkv.reshape(B * T, 3 * D).bfloat16()
    out = torch.empty(B * T, D, device=cuda, dtype=torch.bfloat16)
    lse = torch.empty(B, H, T, device=cuda)
    ops.call("eps_attn_fwd", qkv, out, lse, B, T, H, dh, C.c_float(dh ** -0.5), _s())
    ref, ref_lse = _attn_ref(qkv.float(), B, T, H, dh)
    torch.cuda.synchronize()
    assert torch.isfinite(out.float()).all() and torch.isfinite(lse).all()
    assert _rel(out, ref) < 1e-2
    assert ((lse - ref_lse).abs() / ref_lse.abs().clamp_min(1.0)).max().item() < 1e-3


def test_softmax_xent(cuda):
    B, Cn = 37, 1000
    g = torch.Generator(device=cuda).manual_seed(1)
    z = (torch.randn(B, Cn, device=cuda, generator=g) * 3).bfloat16()
    y = torch.randint(0, Cn, (B,), device=cuda, generator=g)
    dz = torch.empty_like(z)
    loss = torch.zeros(1, device=cuda)
    db = torch.zeros(Cn, device=cuda)
    ops.call("eps_softmax_xent_bias", z, y, dz, loss, db, B, Cn, Cn, C.c_float(1.0 / B), _s())
    zf = z.float().requires_grad_()
    ref = F.cross_entropy(zf, y)
    ref.backward()
    torch.cuda.synchronize()
    assert abs(loss.item() / B - ref.item()) < 1e-3 * abs(ref.item()) + 1e-4
    assert _rel(dz, zf.grad) < 1e-2
    assert _rel(db, zf.grad.sum(0)) < 1e-2


def test_sgd_and_sqnorm(cuda):
    n = 1_000_003
    g = torch.Generator(device=cuda).manual_seed(2)
    p = torch.randn(n + 5, device=cuda, generator=g)[:n].contiguous()
    gr = torch.randn(n, device=cuda, generator=g)
    mom = torch.randn(n, device=cuda, generator=g)
    pb = torch.empty(n, dtype=torch.bfloat16, device=cuda)
    p0, g0, m0 = p.clone(), gr.clone(), mom.clone()
    # segmented sum of squares over 3 segments of the flat buffer
    offs = (C.c_int64 * 4)(0, 100, 500_000, n)
    out = torch.zeros(3, dtype=torch.float64, device=cuda)
    ws = torch.empty(8 * 64, dtype=torch.uint8, device=cuda)
    ops.call("eps_grad_sqnorm_flat", gr, offs, 3, out, ws, ws.numel(), _s())
    torch.cuda.synchronize()
    ref = [float((g0[a:b].double() ** 2).sum()) for a, b in ((0, 100), (100, 500_000),
                                                             (500_000, n))]
    for o, r in zip(out.tolist(), ref):
        assert abs(o - r) <= 1e-9 * r
    out2 = torch.zeros(3, dtype=torch.float64, device=cuda)
    ops.call("eps_grad_sqnorm_flat", gr, offs, 3, out2, ws, ws.numel(), _s())
    torch.cuda.synchronize()
    assert out.tolist() == out2.tolist()  # deterministic
    ops.call("eps_sgd_momentum", p, pb, gr, mom, n, C.c_float(0.1), C.c_float(0.9),
             C.c_float(0.01), _s())
    torch.cuda.synchronize()
    m_ref = 0.9 * m0 + g0 + 0.01 * p0
    p_ref = p0 - 0.1 * m_ref
    assert torch.allclose(mom, m_ref, atol=1e-6)
    assert torch.allclose(p, p_ref, atol=1e-6)
    assert torch.equal(pb, p.bfloat16())
    assert gr.abs().max().item() == 0.0


def test_cache_gather_scatter(cuda):
    n_store, T, d = 50, 197, 768
    g = torch.Generator(device=cuda).manual_seed(3)
    store = torch.zeros(n_store, T, d, dtype=torch.bfloat16, device=cuda)
    src = torch.randn(7, T, d, device=cuda, generator=g).bfloat16()
    ids = torch.tensor([3, 49, 0, 17, 18, 5, 31], device=cuda)
    ops.call("eps_cache_scatter", store, ids, 7, T * d * 2, src, _s())
    dst = torch.empty_like(src)
    ops.call("eps_cache_gather", store, ids, 7, T * d * 2, dst, _s())
    torch.cuda.synchronize()
    assert torch.equal(dst, src)
    assert torch.equal(store[ids], src)
    assert store[1].abs().max().item() == 0
    # background gather (prefetch window): few CTAs, grid-stride; from a pinned
    # host store too (read over the host link)
    for ctas in (1, 3, 8):
        dst2 = torch.empty_like(src)
        ops.call("eps_cache_gather_bg", store, ids, 7, T * d * 2, dst2, ctas, _s())
        torch.cuda.synchronize()
        assert torch.equal(dst2, src)
    host = store.cpu().pin_memory()
    dst3 = torch.empty_like(src)
    ops.call("eps_cache_gather_bg", host, ids, 7, T * d * 2, dst3, 8, _s())
    torch.cuda.synchronize()
    assert torch.equal(dst3, src)


def test_patchify_assemble(cuda):
    from oracle.vit_fp32 import patchify
    B, Cc, S, p, d = 3, 3, 224, 16, 768
    g = torch.Generator(device=cuda).manual_seed(4)
    img = torch.randn(B, Cc, S, S, device=cuda, generator=g)
    out = torch.empty(B * 196, Cc * p * p, dtype=torch.bfloat16, device=cuda)
    ops.call("eps_patchify", img, out, B, Cc, S, p, _s())
    torch.cuda.synchronize()
    ref = patchify(img.cpu(), S, p).reshape(B * 196, -1)
    assert torch.equal(out.cpu(), ref.bfloat16())
    small = torch.randn(B, Cc, 32, 32, device=cuda, generator=g)
    ops.call("eps_patchify", small, out, B, Cc, (32 << 16) | 224, p, _s())
    torch.cuda.synchronize()
    ref = patchify(small.cpu(), 224, p).reshape(B * 196, -1)
    assert torch.equal(out.cpu(), ref.bfloat16())
    tok = torch.randn(B * 196, d, device=cuda, generator=g).bfloat16()
    cls = torch.randn(d, device=cuda, generator=g)
    pos = torch.randn(197, d, device=cuda, generator=g)
    x = torch.empty(B, 197, d, dtype=torch.bfloat16, device=cuda)
    ops.call("eps_vit_assemble", tok, cls, pos, x, B, 197, d, _s())
    torch.cuda.synchronize()
    want = torch.cat([cls.expand(B, 1, d), tok.float().reshape(B, 196, d)], 1) + pos
    assert _rel(x, want) < 1e-2


@pytest.mark.parametrize("B", [3, 67, 400])
def test_assemble_bwd(cuda, B):
    """dpos = sum_b dx, dcls = sum_b dx[:, 0], dtok = dx[:, 1:] (bit copy); the
    B >= 64 launch splits the batch over 8 slices with atomics."""
    d, T = 768, 197
    g = torch.Generator(device=cuda).manual_seed(B)
    dx = torch.randn(B, T, d, device=cuda, generator=g).bfloat16()
    dcls = torch.zeros(d, device=cuda)
    dpos = torch.zeros(T, d, device=cuda)
    dtok = torch.empty(B * (T - 1), d, dtype=torch.bfloat16, device=cuda)
    ops.call("eps_vit_assemble_bwd", dx, dcls, dpos, dtok, B, T, d, _s())
    torch.cuda.synchronize()
    want = dx.double().sum(0)
    assert (dpos.double() - want).abs().max().item() < 1e-4 * max(1.0, B ** 0.5)
    assert (dcls.double() - want[0]).abs().max().item() < 1e-4 * max(1.0, B ** 0.5)
    assert torch.equal(dtok, dx[:, 1:].reshape(-1, d))
