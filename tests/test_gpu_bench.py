"""bench.py on the GPU: the JSON line the driver reads (contract in the task
statement) -- one line, metric/unit/value, timing keys, clocks, e2e with the
copied bytes, roofline with measured peak, cpu_baseline from the compiled
reference, kernel launch count -- on a small workload (cfg2, few steps)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_bench_line_cfg2(esp, gpu):
    r = subprocess.run([sys.executable, "bench.py", "--workload", "cfg2", "--steps", "3",
                        "--warmup", "3", "--cpu-seconds", "0.5"], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "clocks", "e2e", "gpu_launches", "roofline", "cpu_baseline"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("cfg2") and d["config"]["N"] == 32001
    assert d["e2e"]["h2d_bytes_per_step"] == 32001 * 32
    assert d["e2e"]["value"] > 0 and d["e2e"]["value"] < d["value"]
    rf = d["roofline"]
    assert rf["bound"] == "fp64" and 0.0 < rf["frac"] < 1.0 and rf["peak"] > 10.0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-12
    assert d["gpu_launches"] == d["launches_per_step"] * d["steps"] > 0
    cb = d["cpu_baseline"]
    if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libesp_ref.so")):
        assert cb["kind"] == "reference" and cb["value"] > 0 and cb["cores"] >= 1
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    # the energy is the reference's (cfg2 fixture)
    import numpy as np
    g = np.load(os.path.join(ROOT, "tests", "golden", "cfg2_sub.npz"))
    assert abs(d["energy"] - float(g["energy"])) <= 1e-11 * abs(float(g["energy"]))
