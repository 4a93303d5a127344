"""Numerics parity of the sm_100a executors vs the CPU oracles (north_star:
losses, activations and gradients, fp32 accumulation, rtol 1e-2 in bf16
versus the reference's fp32).

Per case, one train step on the device and in oracle/{vit,bert}_fp32.py
under both numerics policies (oracle/numerics.py; harness tests/parity_lib.py):

* loss: device vs FP32 within LOSS_RTOL (1e-2);
* per-layer gradient norms (the freeze test's input): within NORM_RTOL (1e-2);
* every gradient tensor and every residual-stream activation X[l]: the
  device's distance from FP32 is within NOISE_FACTOR x the distance of a
  perfect bf16-storage emulation from FP32 (+ NOISE_FLOOR).  A per-tensor
  1e-2 vs FP32 is not attainable by any bf16-storage design at these depths
  (the emulation itself sits at 1.0-1.5 % for ViT-B/16 and 2-4 % for BERT;
  measured table and the rounding-chaos experiment in
  profiles/r02/numerics.md);
* mathematically-zero gradients (QA span head: classifier bias, final LN
  bias): no larger than the emulation's rounding noise (x 3);
* frozen tensors: exactly zero;
* 10-step SGD-momentum loss trajectories: every step within TRAJ_RTOL (1e-2).

Cases follow VERDICT r01 "next round" 1: ViT-B/16 at batch >= 8 with
L_f in {0, 6}, BERT-base-384, BERT-large-128 (plus the tiny configs and the
CIFAR-shaped ViT, micro-batched and frozen variants).
"""
import pytest

from tests.parity_lib import (LOSS_RTOL, NOISE_FACTOR, NOISE_FLOOR, NORM_RTOL, TRAJ_RTOL,
                              run_case, trajectory)

pytestmark = pytest.mark.gpu

CASES = [
    ("tiny-vit", 16, 0, 1),
    ("tiny-vit", 16, 2, 3),
    ("vit-b16", 8, 0, 1),
    ("vit-b16", 8, 6, 2),
    ("vit-b16-cifar100", 4, 4, 1),
    ("tiny-bert-qa", 4, 0, 1),
    ("tiny-bert-qa", 5, 1, 2),
    ("tiny-bert-cls", 6, 1, 3),
    ("bert-base-384", 4, 0, 1),
    ("bert-base-384", 4, 6, 2),
    ("bert-large-128", 8, 0, 1),
    ("bert-large-128", 8, 12, 2),
]


@pytest.mark.parametrize("cfg,batch,l_frozen,micro", CASES)
def test_step_numerics(cuda, cfg, batch, l_frozen, micro):
    c = run_case(cfg, batch, l_frozen, micro)
    assert abs(c.loss["dev"] - c.loss["fp32"]) <= LOSS_RTOL * abs(c.loss["fp32"]), c.loss
    assert not c.frozen_nonzero, c.frozen_nonzero
    bad = {n: v for n, v in c.grads.items()
           if v["vs_fp32"] > NOISE_FACTOR * v["intrinsic"] + NOISE_FLOOR}
    assert not bad, bad
    for l, v in enumerate(c.acts):
        assert v["vs_fp32"] <= NOISE_FACTOR * v["intrinsic"] + NOISE_FLOOR, (l, v)
    for l, v in enumerate(c.norms):
        if l < l_frozen:
            assert v["dev"] == 0.0
        else:
            assert v["vs_fp32"] <= NORM_RTOL, (l, v)
    for n, ratio in c.zero_tensors.items():
        assert ratio <= 3.0, (n, ratio)


@pytest.mark.parametrize("cfg,batch,l_frozen,lr", [
    ("vit-b16", 8, 0, 5e-4),
    ("vit-b16", 8, 6, 1e-3),
    ("bert-base-384", 4, 0, 5e-4),
    ("bert-large-128", 8, 0, 1e-3),
])
def test_loss_trajectory(cuda, cfg, batch, l_frozen, lr):
    """10 SGD-momentum steps on one batch: the device's loss curve tracks the
    fp32 oracle's at every step."""
    dev, ref = trajectory(cfg, batch, 10, lr, l_frozen=l_frozen)
    assert ref[-1] < 0.8 * ref[0]  # the trajectory actually moves
    for step, (a, r) in enumerate(zip(dev, ref)):
        assert abs(a - r) <= TRAJ_RTOL * abs(r), (step, dev, ref)
