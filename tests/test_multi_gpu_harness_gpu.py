"""The multi-GPU sweep harness (tools/multi_gpu_sweeps.py: SURVEY.md 8(f)
rows 3-4 -- feature ladder, transition overheads, chunks sweep at K = N)
stays runnable: one torchrun rank on cuda:0 with the tiny ViT; a multi-GPU
box runs the same command with --nproc-per-node N."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_harness_one_rank(cuda, tmp_path):
    out = tmp_path / "sweeps.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           "1", "--master-addr", "127.0.0.1", "--master-port", "29561",
           os.path.join(ROOT, "tools/multi_gpu_sweeps.py"), "tiny-vit", "2", "4", str(out)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.load(open(out))
    assert d["world"] == 1
    assert [x["rung"] for x in d["ladder"]] == ["baseline", "freeze", "autopipe",
                                                "autopipe+autocache", "autopipe+autodp", "all"]
    assert all(x["measured_total_s"] > 0 for x in d["ladder"])
    assert len(d["transitions"]) == 4
    assert d["chunks_sweep"] and all(x["measured_iteration_s"] > 0 for x in d["chunks_sweep"])
