"""bench.py plumbing on the CPU container: the reference arm (compiled
reference, oracle/_ref) must not load this repo's CUDA library, must print
the same `config` as the GPU arm would, and `--gpus N` must launch N ranks
itself (torch.distributed.run) with rank 0 printing n_gpus = N."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

REF_SO = os.path.join(ROOT, "oracle", "_ref", "libesp_ref.so")
pytestmark = pytest.mark.skipif(not os.path.exists(REF_SO), reason="oracle/_ref not built")

_PROBE = r"""
import runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--workload", "cfg1", "--steps", "1"]
try:
    runpy.run_path("bench.py", run_name="__main__")
except SystemExit:
    pass
maps = open("/proc/self/maps").read()
print("LOADED_OURS=%d" % ("libesp_b200.so" in maps))
print("LOADED_REF=%d" % ("libesp_ref.so" in maps))
print("PKG_IMPORTED=%d" % ("paper_2505_09727_b200" in sys.modules))
"""


def _json_line(out):
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


def test_reference_arm_loads_only_the_reference():
    r = subprocess.run([sys.executable, "-c", _PROBE], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    line = _json_line(r.stdout)
    assert line["impl"] == "reference" and line["n_gpus"] == 1
    assert "LOADED_OURS=0" in r.stdout and "LOADED_REF=1" in r.stdout
    assert "PKG_IMPORTED=0" in r.stdout


def test_reference_config_matches_gpu_arm_keys():
    sys.path.insert(0, ROOT)
    import bench
    S = bench.load_systems()
    c = S.config("cfg5")
    cfg = bench.bench_config(c, c.N, (c.L,) * 3, (180, 180, 180), 6, "ik", "replicas", 1)
    assert set(cfg) == {"workload", "N", "box_L", "r_c", "eps", "nf", "P", "force_method",
                        "parallelism", "l2"}
    assert cfg["parallelism"] == "single GPU"


def test_gpus_flag_spawns_ranks():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "cfg1",
                        "--gpus", "2", "--steps", "1"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600, env=env)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "replicas x2"
