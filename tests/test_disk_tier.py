"""AutoCache disk tier (csrc/runtime/disk_tier.cpp) on the CPU: the host side
of the reference's CacheTierSim (autocache.cpp:69-150) executed for real --
rows written by sample id come back bit-exact in any per-epoch order through
the sliding window; batches beyond the window are refused until earlier ones
are released; block prefetch / eviction counts follow CacheTierSim."""
import os

import pytest
import torch

from paper_2102_03161_b200.disk_tier import DiskTier, DiskTierError

ROW = 302_592  # one ViT-B/16 boundary activation (197 x 768 bf16)


def _rows(n, row_bytes, seed):
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, 256, (n, row_bytes), generator=g, dtype=torch.uint8)


@pytest.mark.parametrize("row_bytes,batch,block,window", [(ROW, 4, 2, 4), (1000, 3, 1, 2),
                                                          (4096, 5, 3, 3)])
def test_roundtrip_shuffled_epochs(tmp_path, row_bytes, batch, block, window):
    n = 37  # ragged last batch and block
    data = _rows(n, row_bytes, 1)
    t = DiskTier(str(tmp_path / "cache.bin"), n, row_bytes, batch, block_batches=block,
                 window_batches=window, threads=4)
    assert t.stride % 4096 == 0 and t.stride >= row_bytes
    # written in two halves, out of order
    ids = torch.randperm(n, generator=torch.Generator().manual_seed(2))
    t.write(ids[:20], data[ids[:20]])
    t.write(ids[20:], data[ids[20:]])
    for epoch in range(3):
        order = torch.randperm(n, generator=torch.Generator().manual_seed(10 + epoch))
        t.begin_epoch(order)
        nb = -(-n // batch)
        for b in range(nb):
            view, stall = t.batch_view(b)
            assert stall >= 0.0
            want = data[order[b * batch:(b + 1) * batch]]
            assert view.shape[0] == want.shape[0]
            assert torch.equal(view[:, :row_bytes], want)
            t.release(b)
        s = t.stats()
        blocks = -(-nb // block)
        assert s["prefetches"] == blocks * (epoch + 1)
        assert s["evictions"] == blocks * (epoch + 1)
        assert s["max_resident_bytes"] <= (window // block) * block * batch * t.stride
    assert s["bytes_written"] >= n * row_bytes
    t.close()


def test_window_bounds(tmp_path):
    n, row_bytes, batch = 16, 512, 2
    t = DiskTier(str(tmp_path / "c.bin"), n, row_bytes, batch, block_batches=2,
                 window_batches=2, threads=2)
    data = _rows(n, row_bytes, 3)
    t.write(torch.arange(n), data)
    t.begin_epoch(torch.arange(n))
    t.acquire(0)
    t.acquire(1)
    with pytest.raises(DiskTierError):  # block 1 is outside the one-block window
        t.acquire(2)
    t.release(0)
    t.release(1)  # block 0 consumed: evicted, block 1 issued
    view, _ = t.batch_view(2)
    assert torch.equal(view[:, :row_bytes], data[4:6])
    with pytest.raises(DiskTierError):  # evicted
        t.acquire(0)
    with pytest.raises(DiskTierError):  # beyond the epoch
        t.acquire(8)
    t.close()


def test_invalid_arguments(tmp_path):
    with pytest.raises(DiskTierError):
        DiskTier(str(tmp_path / "x.bin"), 4, 100, 2, block_batches=4, window_batches=2)
    t = DiskTier(str(tmp_path / "y.bin"), 4, 100, 2, block_batches=1, window_batches=2)
    with pytest.raises(DiskTierError):
        t.write(torch.tensor([4]), torch.zeros(1, 100, dtype=torch.uint8))
    with pytest.raises(DiskTierError):
        t.begin_epoch([0, 5])
    t.close()
    assert os.path.getsize(tmp_path / "y.bin") == 4 * 4096


def test_explicit_uneven_batches(tmp_path):
    n, row_bytes = 23, 700
    data = _rows(n, row_bytes, 5)
    t = DiskTier(str(tmp_path / "u.bin"), n, row_bytes, 6, block_batches=2, window_batches=4)
    t.write(torch.arange(n), data)
    order = torch.randperm(n, generator=torch.Generator().manual_seed(7))
    sizes = [6, 6, 6, 5]  # microbatch_offsets-style: remainder on the leading batches
    offs = [sum(sizes[:i]) for i in range(len(sizes))]
    t.begin_epoch(order, list(zip(offs, sizes)))
    for b, (o, sz) in enumerate(zip(offs, sizes)):
        view, _ = t.batch_view(b)
        assert view.shape[0] == sz
        assert torch.equal(view[:, :row_bytes], data[order[o:o + sz]])
        t.release(b)
    with pytest.raises(DiskTierError):  # a batch larger than batch_rows
        t.begin_epoch(order, [(0, 7), (7, 16)])
    t.close()
