"""The native epoch loop (csrc/runtime/trainer.cpp, eps_trainer_*) against
the Python Trainer on the same GPU, parameters and data: identical decisions
every epoch (freeze count, K / R / M, AutoCache state), the same losses and
gradient norms up to fp32 reduction order; with the scenario's synthetic
norms it follows the reference's golden decisions; the eps_train CLI runs a
scenario file end to end."""
import json
import os
import subprocess

import pytest
import torch

from oracle import eps_oracle as O
from paper_2102_03161_b200 import configs
from paper_2102_03161_b200.native_trainer import NativeTrainer
from paper_2102_03161_b200.trainer import Trainer

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests/golden/decisions.json")))


def _scenario(alpha=None, epochs=6, batch=16):
    s = configs.scenario("tiny-vit", 1)
    s["training"]["per_pipeline_batch"] = batch
    s["training"]["epochs"] = epochs
    if alpha is not None:
        s["training"]["alpha"] = alpha
    return s


@pytest.mark.parametrize("alpha,batch,iters", [(None, 16, 3), (0.5, 24, 2)])
def test_native_matches_python_trainer(cuda, alpha, batch, iters):
    scen = _scenario(alpha, epochs=6, batch=batch)
    g = configs.GEOMETRIES["tiny-vit"]
    py = Trainer(scen, g, iterations_per_epoch=iters, device_norms=True, lr=0.05)
    p0 = py.ex.p32.detach().clone()
    nat = NativeTrainer(scen, g, iterations_per_epoch=iters, lr=0.05, init_params=p0,
                        images=py.images, labels=py.labels)
    rows_py = py.run(6)
    rows_nat = nat.run(6)
    nat.close()
    frozen = set()
    for a, b in zip(rows_py, rows_nat):
        assert (a.epoch, a.l_frozen, a.k, a.r, a.m, a.cache_enabled, a.cache_moved) == (
            b.epoch, b.l_frozen, b.k, b.r, b.m, b.cache_enabled, b.cache_moved)
        assert abs(a.mean_loss - b.mean_loss) <= 1e-3 * abs(a.mean_loss)
        na, nb = torch.tensor(a.norms), torch.tensor(b.norms)
        assert ((na - nb).norm() / na.norm()).item() < 1e-2
        assert b.samples == a.samples and b.throughput_sps > 0
        frozen.add(b.l_frozen)
    assert len(frozen) > 1  # the run froze layers (and exercised the cache modes)
    # the native run's freeze decisions are the reference algorithm's on its own norms
    st = O.FreezeState(scen["training"]["alpha"])
    for e in range(1, len(rows_nat)):
        assert O.next_frozen_count(st, rows_nat[e - 1].norms, g.layers) == rows_nat[e].l_frozen


def test_native_follows_golden_decisions(cuda):
    case = next(c for c in GOLDEN["scenarios"] if c["name"] == "tiny-vit-g1")
    scen = json.loads(json.dumps(case["scenario"]))
    scen["training"]["per_pipeline_batch"] = 16
    nat = NativeTrainer(scen, configs.GEOMETRIES["tiny-vit"], iterations_per_epoch=2,
                        device_norms=False)
    rows = nat.run(6)
    nat.close()
    for r, want in zip(rows, case["rows"]):
        assert (r.l_frozen, r.k, r.r, r.m, int(r.cache_enabled)) == (
            want["l_frozen"], want["pipeline_length"], want["replica_width"],
            want["micro_batches"], want["cache_enabled"])
        assert r.mean_loss == r.mean_loss and abs(r.mean_loss) < 1e6


def test_cli_runs_scenario_file(cuda, tmp_path):
    subprocess.run(["make", "-C", ROOT, "train"], check=True, capture_output=True)
    scen = tmp_path / "s.json"
    scen.write_text(json.dumps(_scenario(alpha=0.5, epochs=4)))
    out = tmp_path / "run.csv"
    r = subprocess.run([os.path.join(ROOT, "build", "eps_train"), "--scenario", str(scen),
                        "--geometry", "tiny-vit", "--iterations", "3", "--epochs", "4",
                        "--csv", str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0].startswith("epoch,l_frozen,k,r,m,") and len(lines) == 5
    rows = [l.split(",") for l in lines[1:]]
    assert [int(x[0]) for x in rows] == [0, 1, 2, 3]
    assert all(float(x[7]) > 0 for x in rows)  # throughput
    assert "loss" in r.stderr


# ---- BERT (configs 4 / 5 family) through the same native loop ----------------------
def _bert_scenario(geo_name, batch=16, epochs=5, alpha=0.5):
    g = configs.GEOMETRIES[geo_name]
    s = configs.scenario("bert-large-128", 1)
    s["model"] = dict(name=geo_name, bytes_per_param=4, **configs.model_spec(g))
    s["training"]["per_pipeline_batch"] = batch
    s["training"]["epochs"] = epochs
    s["training"]["alpha"] = alpha
    return s, g


@pytest.mark.parametrize("geo_name", ["tiny-bert-qa", "tiny-bert-cls"])
def test_native_bert_first_iteration_matches_executor(cuda, geo_name):
    """One iteration per epoch: the native loop's epoch-0 loss is the BERT
    executor's train_step loss on the same batch (the epoch's first shard ids:
    token / segment gathers and the SQuAD start | end label layout line up)."""
    from paper_2102_03161_b200 import bert
    from paper_2102_03161_b200.capi import ClusterSpec, EpsApi
    from paper_2102_03161_b200 import LIB_PATH
    scen, g = _bert_scenario(geo_name, batch=16)
    N, T = 16, g.tokens
    gen = torch.Generator(device=cuda).manual_seed(5)
    tok = torch.randint(0, g.vocab, (N, T), device=cuda, generator=gen)
    seg = torch.zeros(N, T, dtype=torch.int64, device=cuda)
    seg[:, T // 2:] = 1
    lab = (torch.randint(0, T, (2, N), device=cuda, generator=gen) if g.head == "qa" else
           torch.randint(0, g.classes, (N,), device=cuda, generator=gen))
    ex = bert.BertExecutor(g, max_batch=N, seed=11)
    p0 = ex.p32.detach().clone()
    nat = NativeTrainer(scen, g, iterations_per_epoch=1, lr=0.05, seed=17, init_params=p0,
                        images=torch.stack([tok, seg]).contiguous(), labels=lab.contiguous())
    r0 = nat.run_epoch(0)
    nat.close()
    api = EpsApi(LIB_PATH, "eps_")
    _, shards = api.redistribute(N, ClusterSpec(1, 1), 1, 0, 17)
    ids = torch.tensor(shards[0], device=cuda)
    x = torch.stack([tok[ids], seg[ids]]).contiguous()
    y = (torch.cat([lab[0][ids], lab[1][ids]]) if g.head == "qa" else lab[ids]).contiguous()
    loss = ex.train_step(x, y).item() / N
    assert abs(loss - r0.mean_loss) <= 2e-3 * abs(loss), (loss, r0.mean_loss)


@pytest.mark.parametrize("geo_name", ["tiny-bert-qa", "tiny-bert-cls"])
def test_native_bert_device_norm_decisions(cuda, geo_name):
    scen, g = _bert_scenario(geo_name, batch=16, epochs=5)
    nat = NativeTrainer(scen, g, iterations_per_epoch=3, lr=0.05)
    rows = nat.run(5)
    nat.close()
    st = O.FreezeState(scen["training"]["alpha"])
    for e in range(len(rows)):
        assert rows[e].mean_loss == rows[e].mean_loss and rows[e].throughput_sps > 0
        assert len(rows[e].norms) == g.layers and all(n >= 0 for n in rows[e].norms)
        if e > 0:
            assert O.next_frozen_count(st, rows[e - 1].norms, g.layers) == rows[e].l_frozen


def test_cli_runs_bert_scenario(cuda, tmp_path):
    subprocess.run(["make", "-C", ROOT, "train"], check=True, capture_output=True)
    scen, _ = _bert_scenario("tiny-bert-cls", batch=16, epochs=3)
    f = tmp_path / "s.json"
    f.write_text(json.dumps(scen))
    r = subprocess.run([os.path.join(ROOT, "build", "eps_train"), "--scenario", str(f),
                        "--geometry", "tiny-bert-cls", "--iterations", "2", "--epochs", "3"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    rows = r.stdout.strip().splitlines()
    assert rows[0].startswith("epoch,l_frozen") and len(rows) == 4
