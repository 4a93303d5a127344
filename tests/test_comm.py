"""The communicator plane behind the C ABI (eps_comm_* / eps_allreduce* /
eps_broadcast / eps_p2p_*, csrc/runtime/comm.cpp).

CPU: NCCL resolves at run time and hands out a unique id (no device needed).
GPU (one B200, so one rank): world communicator, ncclCommSplit children with
and without a color, ncclAvg / sum / max all-reduces, broadcast, and a
grouped send / receive pair to self -- every call stream-ordered on the
current stream.  Multi-rank NCCL needs one GPU per rank (NCCL rejects two
ranks on one device); those paths are exercised on a multi-GPU box by
`bench.py --gpus N` (EpsTransport).
"""
import pytest
import torch

from paper_2102_03161_b200 import comm


def test_nccl_resolves_and_creates_unique_id():
    assert comm.nccl_version() >= 21000  # ncclAvg / ncclCommSplit era
    a, b = comm.unique_id(), comm.unique_id()
    assert len(a) == 128 and a != b


@pytest.mark.gpu
def test_world_of_one(cuda):
    w = comm.Comm.world(0, 1, uid=comm.unique_id())
    assert (w.rank, w.size) == (0, 1)
    x = torch.arange(1, 1001, dtype=torch.float32, device=cuda)
    ref = x.clone()
    w.all_reduce_bucket(x, average=True)   # mean over one replica = identity
    w.all_reduce(x, comm.OP_SUM)
    w.all_reduce(x, comm.OP_MAX)
    d = torch.tensor([2.5, -1.0], dtype=torch.float64, device=cuda)
    w.all_reduce(d, comm.OP_SUM)
    bf = torch.ones(64, dtype=torch.bfloat16, device=cuda)
    w.broadcast(bf, 0)
    src = torch.randn(4096, device=cuda)
    dst = torch.zeros_like(src)
    w.group_start()
    w.send(src, 0)
    w.recv(dst, 0)
    w.group_end()
    child = w.split(3, 0)
    assert child is not None and (child.rank, child.size) == (0, 1)
    child.all_reduce_bucket(x, average=True)
    torch.cuda.synchronize()
    assert torch.equal(x, ref)
    assert torch.equal(d.cpu(), torch.tensor([2.5, -1.0], dtype=torch.float64))
    assert torch.equal(dst, src)
    child.free()
    w.free()


@pytest.mark.gpu
def test_errors_are_statuses(cuda):
    w = comm.Comm.world(0, 1, uid=comm.unique_id())
    x = torch.zeros(8, device=cuda)
    with pytest.raises(RuntimeError):
        w.send(x, 3)  # no such peer: EPS_EINVAL, not a crash
    w.free()
