"""Native training loop (csrc/runtime/trainer.cpp) -- the host-side checks that
need no GPU: the C entry points are exported, a multi-GPU scenario is refused
before any device work with a readable error, and the eps_train CLI builds and
validates its arguments."""
import ctypes as C
import json
import os
import subprocess

from paper_2102_03161_b200 import configs, ops
from paper_2102_03161_b200.capi import EpsApi, Scenario
from paper_2102_03161_b200.vit import geom_array
from paper_2102_03161_b200 import LIB_PATH

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_trainer_refuses_multi_gpu_cluster():
    api = EpsApi(LIB_PATH, "eps_")
    lib = ops.api().lib
    f = lib.eps_trainer_create
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_uint64, C.c_float, C.c_float,
                  C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    sc = Scenario(api, configs.scenario("tiny-vit", 8))
    h = C.c_void_p()
    rc = f(sc.h, 0, geom_array(configs.GEOMETRIES["tiny-vit"], 64), 2, 17, 1e-3, 0.9, 1, None,
           None, None, C.byref(h))
    assert rc == 1 and not h.value  # EPS_EINVAL
    lib.eps_last_error.restype = C.c_char_p
    assert b"one GPU" in lib.eps_last_error()


def test_cli_builds_and_validates_arguments(tmp_path):
    subprocess.run(["make", "-C", ROOT, "train"], check=True, capture_output=True)
    exe = os.path.join(ROOT, "build", "eps_train")
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 2 and "usage" in r.stderr
    scen = tmp_path / "s.json"
    scen.write_text(json.dumps(configs.scenario("tiny-vit", 8)))
    r = subprocess.run([exe, "--scenario", str(scen), "--geometry", "tiny-vit", "--iterations",
                        "2"], capture_output=True, text=True)
    assert r.returncode == 1 and "one GPU" in r.stderr
