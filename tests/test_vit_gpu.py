"""ViT executor properties on the sm_100a path: AutoCache gather / scatter
equivalence, host-tier store, SGD, and the full-size (batch 400) step.
Per-tensor numerics parity vs the CPU oracles lives in test_numerics_gpu.py.
"""
import pytest
import torch

from oracle import vit_fp32
from paper_2102_03161_b200.configs import GEOMETRIES, Geometry
from paper_2102_03161_b200.vit import VitExecutor, init_params

pytestmark = pytest.mark.gpu

LOSS_RTOL = 1e-2


def _rel(a, b):
    return ((a.float().cpu() - b.float().cpu()).norm() / (b.float().cpu().norm() + 1e-12)).item()


def _data(g: Geometry, batch: int, seed: int):
    gen = torch.Generator().manual_seed(seed)
    images = torch.randn(batch, g.channels, g.input_image, g.input_image, generator=gen)
    labels = torch.randint(0, g.classes, (batch,), generator=gen)
    return images, labels


def test_cache_paths_equivalent(cuda):
    """AutoCache: gathering X[L_f] from the HBM store == recomputing the frozen
    prefix; a boundary move forwards the delta once and writes the store."""
    g = GEOMETRIES["tiny-vit"]
    batch, lf = 8, 2
    params = init_params(g, seed=3)
    images, labels = _data(g, batch, seed=9)
    images, labels = images.cuda(), labels.cuda()
    store = torch.zeros(32, g.tokens, g.hidden, dtype=torch.bfloat16, device=cuda)
    ids = torch.tensor([5, 1, 30, 7, 8, 2, 0, 19], device=cuda)

    ex = VitExecutor(g, max_batch=batch, params=params)
    base = ex.train_step(images, labels, l_frozen=lf).item()
    g_base = ex.g32.clone()
    ex.g32.zero_()
    # epoch where the boundary moves 0 -> 2: recompute, scatter X[2]
    moved = ex.train_step(images, labels, l_frozen=lf, cache_mode=2, cache_old=0, store=store,
                          ids=ids).item()
    torch.cuda.synchronize()
    want = ex.boundary_activation(lf, batch).clone()
    assert torch.equal(store[ids], want)
    g_moved = ex.g32.clone()
    ex.g32.zero_()
    # steady state: gather X[2], skip the frozen prefix entirely
    cached = ex.train_step(images, labels, l_frozen=lf, cache_mode=1, store=store, ids=ids).item()
    torch.cuda.synchronize()
    assert abs(moved - base) <= 1e-5 * abs(base)
    assert abs(cached - base) <= 1e-5 * abs(base)
    assert _rel(g_moved, g_base) < 1e-5
    assert _rel(ex.g32, g_base) < 1e-5
    # trailing boundary (runner.cpp:186-213): the store stays at X[2] while
    # L_f = 3 -- gather X[2], forward layer 2, write nothing
    before = store.clone()
    ex.g32.zero_()
    trail = ex.train_step(images, labels, l_frozen=3, cache_mode=3, cache_old=2, store=store,
                          ids=ids).item()
    g_trail = ex.g32.clone()
    ex.g32.zero_()
    ref3 = ex.train_step(images, labels, l_frozen=3).item()
    torch.cuda.synchronize()
    assert torch.equal(store, before)
    assert abs(trail - ref3) <= 1e-5 * abs(ref3)
    assert _rel(g_trail, ex.g32) < 1e-5
    # boundary move 2 -> 3 reads the old boundary from the store
    ex.g32.zero_()
    ex.train_step(images, labels, l_frozen=3, cache_mode=2, cache_old=2, store=store, ids=ids)
    torch.cuda.synchronize()
    assert torch.equal(store[ids], ex.boundary_activation(3, batch))


def test_sgd_step_and_loss_decreases(cuda):
    g = GEOMETRIES["tiny-vit"]
    batch = 32
    ex = VitExecutor(g, max_batch=batch, seed=1)
    images, labels = _data(g, batch, seed=2)
    images, labels = images.cuda(), labels.cuda()
    losses = []
    for _ in range(8):
        losses.append(ex.train_step(images, labels).item() / batch)
        ex.sgd(0, lr=0.05)
    torch.cuda.synchronize()
    assert losses[-1] < losses[0] - 0.1, losses
    assert ex.g32.abs().max().item() == 0.0  # optimizer consumed the grads


def test_cache_host_tier(cuda):
    """AutoCache host tier: the store in pinned host
    memory, read and written by the same gather / scatter kernels over the
    host link (UVA), gives the same step as the HBM store."""
    g = GEOMETRIES["tiny-vit"]
    batch, lf = 8, 2
    params = init_params(g, seed=3)
    images, labels = _data(g, batch, seed=9)
    images, labels = images.cuda(), labels.cuda()
    ids = torch.tensor([5, 1, 30, 7, 8, 2, 0, 19], device=cuda)
    dev_store = torch.zeros(32, g.tokens, g.hidden, dtype=torch.bfloat16, device=cuda)
    host_store = torch.zeros(32, g.tokens, g.hidden, dtype=torch.bfloat16).pin_memory()
    ex = VitExecutor(g, max_batch=batch, params=params)
    ex.train_step(images, labels, l_frozen=lf, cache_mode=2, store=dev_store, ids=ids)
    ex.train_step(images, labels, l_frozen=lf, cache_mode=2, store=host_store, ids=ids)
    torch.cuda.synchronize()
    assert torch.equal(host_store, dev_store.cpu())
    ex.g32.zero_()
    a = ex.train_step(images, labels, l_frozen=lf, cache_mode=1, store=dev_store, ids=ids).item()
    ga = ex.g32.clone()
    ex.g32.zero_()
    b = ex.train_step(images, labels, l_frozen=lf, cache_mode=1, store=host_store, ids=ids).item()
    torch.cuda.synchronize()
    assert abs(a - b) <= 1e-6 * abs(a)  # loss sum uses fp32 atomics
    assert torch.allclose(ga, ex.g32, rtol=1e-5, atol=1e-7)


def test_full_size_step_properties(cuda):
    """BASELINE config 2 at full size (ViT-B/16, batch 400 -- 78,800 token rows,
    CTA-pair GEMM tiles with a partial last pair, every attention / LN path):
    size-independent properties instead of a CPU oracle at this size.
    (1) micro-batch invariance (GPipe's contract): one pass == 5 micro-batches
    (different GEMM / attention tilings) for the loss and every gradient;
    (2) additivity: the loss sum of the batch == the sums of its two halves;
    (3) its first 4 samples alone match the fp32 oracle."""
    g = GEOMETRIES["vit-b16"]
    batch = 400
    params = init_params(g, seed=23)
    images, labels = _data(g, batch, seed=9)
    x, y = images.cuda(), labels.cuda()
    ex = VitExecutor(g, max_batch=batch, params=params)
    loss1 = ex.train_step(x, y, micro_batches=1).item()
    g1 = ex.g32.clone()
    ex.g32.zero_()
    loss5 = ex.train_step(x, y, micro_batches=5).item()
    torch.cuda.synchronize()
    assert abs(loss5 - loss1) <= 1e-3 * abs(loss1)
    assert _rel(ex.g32, g1) < 1e-2
    assert torch.isfinite(g1).all()
    halves = 0.0
    for lo in (0, 200):
        ex.g32.zero_()
        halves += ex.train_step(x[lo:lo + 200], y[lo:lo + 200]).item()
    assert abs(halves - loss1) <= 1e-3 * abs(loss1)
    ref_loss, _, _ = vit_fp32.train_step(params, images[:4], labels[:4], g, 0)
    ex.g32.zero_()
    l4 = ex.train_step(x[:4], y[:4]).item() / 4
    assert abs(l4 - ref_loss.item()) <= LOSS_RTOL * abs(ref_loss.item())
