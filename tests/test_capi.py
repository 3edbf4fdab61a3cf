"""C-ABI boundary: the library loads, exports every symbol include/esp_b200.h
declares, and maps errors like the reference; host-side helpers."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "esp_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(esp_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(esp):
    lib = ctypes.CDLL(esp.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_no_cpu_fallback(esp):
    """A host-only plan refuses device work instead of computing on the CPU."""
    p = esp.build_plan((10.0, 10.0, 10.0), "pswf", 1e-3, 1.0, device=-1)
    sysm = esp.ParticleSystem((10.0, 10.0, 10.0), np.array([1.0, -1.0]),
                              np.array([[1.0, 1.0, 1.0], [2.0, 2.0, 2.0]]))
    with pytest.raises(esp.CudaError):
        esp.evaluate(p, sysm)
    with pytest.raises(esp.CudaError):
        esp.local_sum(p, sysm)
    if esp.device_count() == 0:
        with pytest.raises(esp.CudaError):
            esp.build_plan((10.0, 10.0, 10.0), "pswf", 1e-3, 1.0, device=0)


def test_require_neutral(esp):
    ok = esp.ParticleSystem((1, 1, 1), np.array([1.0, -1.0]), np.zeros((2, 3)))
    esp.require_neutral(ok)
    bad = esp.ParticleSystem((1, 1, 1), np.array([1.0, -0.5]), np.zeros((2, 3)))
    with pytest.raises(esp.NumericalError):
        esp.require_neutral(bad)


def test_unknown_family_and_force_method(esp):
    with pytest.raises(esp.InvalidArgument):
        esp.build_plan((10, 10, 10), "ewald", 1e-4, 1.0, device=-1)
    with pytest.raises(esp.InvalidArgument):
        esp.build_plan((10, 10, 10), "pswf", 1e-4, 1.0, esp.Overrides(force_method="xx"),
                       device=-1)


def test_generators_match_reference_stream():
    """io.hpp:33-44, 82-148: bit-identical seeded systems."""
    from oracle import esp_oracle as O
    from paper_2505_09727_b200 import systems as S
    for N, box, seed in [(1000, (10.0, 10.0, 10.0), 1), (64, (10.0, 10.0, 10.5), 17)]:
        p1, q1 = S.generate_system("random", N, box, seed)
        p2, q2 = O.random_system(N, box, seed)
        assert np.array_equal(p1, p2) and np.array_equal(q1, q2)
    from oracle import ref
    if ref.available():
        for kind, N, box in [("random", 100, (3.0, 4.0, 5.0)), ("rocksalt", 8, (2.0,) * 3),
                             ("water-like", 81, (9.0,) * 3)]:
            p1, q1 = S.generate_system(kind, N, box, 5)
            p2, q2 = ref.generate(kind, N, box, 5)
            assert np.array_equal(p1, p2) and np.array_equal(q1, q2)


def test_water_box_geometry():
    from paper_2505_09727_b200 import systems as S
    pos, q, L = S.water_box(1000, seed=3)
    assert abs(L - (1000 / 0.0334) ** (1 / 3)) < 1e-12
    assert q.sum() == 0.0 and pos.min() >= 0.0 and pos.max() < L
    o, h1, h2 = pos[0::3], pos[1::3], pos[2::3]

    def mi(d):
        return d - L * np.round(d / L)
    d1, d2 = mi(h1 - o), mi(h2 - o)
    np.testing.assert_allclose(np.linalg.norm(d1, axis=1), 1.0, atol=1e-12)
    np.testing.assert_allclose(np.linalg.norm(d2, axis=1), 1.0, atol=1e-12)
    ang = np.degrees(np.arccos(np.einsum("ij,ij->i", d1, d2)))
    np.testing.assert_allclose(ang, 109.47, atol=1e-9)


def test_particles_file_round_trip(tmp_path):
    from paper_2505_09727_b200 import systems as S
    pos, q = S.generate_system("random", 50, (3.0, 4.0, 5.0), 9)
    f = tmp_path / "particles.txt"
    S.write_particles(str(f), pos, q, (3.0, 4.0, 5.0))
    p2, q2, box = S.read_particles(str(f))
    assert box == (3.0, 4.0, 5.0)
    assert np.array_equal(p2, pos) and np.array_equal(q2, q)


def test_plan_info_layout_matches_the_header():
    """The ctypes mirror of esp_plan_info / esp_pencil_info reads the values
    the C side wrote (a field-order slip shows up as shuffled values)."""
    import paper_2505_09727_b200 as esp
    box = (50.0, 44.0, 47.0)
    p = esp.build_plan(box, "pswf", 1e-4, 8.0, device=-1)
    assert p.box == box
    assert all(abs(p.h[d] - box[d] / p.nf[d]) < 1e-12 for d in range(3))
    assert p.r_c == 8.0 and p.eps == 1e-4 and p.P >= 3
    assert all(n >= d for n, d in zip(p.nf, p.base_nf))
    g = esp.pencil_geometry(p, 1, 2)
    assert g["nf"] == p.nf and g["rank"] == 1 and g["nranks"] == 2
    assert abs(g["hx"] - p.h[0]) < 1e-15 and g["x1"] == p.nf[0]
    assert g["slab_reals"] == (g["x1"] - g["x0"] + 2 * g["halo"]) * p.nf[1] * p.nf[2]


def test_shard_owner_matches_pencil_geometry(esp):
    """esp_shard_owner: the rank whose planes hold clamp(floor(fold(x)/hx)),
    the same ownership rule as the distributed FFT (esp_pencil_geometry)."""
    from paper_2505_09727_b200 import systems as S
    c = S.config("cfg2")
    pos, q, box = c.system()
    p = esp.build_plan(box, "pswf", c.eps, c.r_c, device=-1)
    for G in (2, 3, 4):
        own = esp.shard_owner(p, G, pos - box[0] * 0.5)  # unfolded images
        geo = [esp.pencil_geometry(p, r, G) for r in range(G)]
        x = np.mod(pos[:, 0] - box[0] * 0.5, box[0])
        pl = np.clip(np.floor(x / geo[0]["hx"]).astype(int), 0, p.nf[0] - 1)
        want = np.searchsorted([g["x1"] for g in geo], pl, side="right")
        assert np.array_equal(own, want)
        assert np.bincount(own, minlength=G).min() > 0


def test_shard_needs_a_device_plan(esp):
    p = esp.build_plan((40.0, 40.0, 40.0), "pswf", 1e-3, 4.0, device=-1)
    with pytest.raises(esp.CudaError):
        esp.Shard(p, 0, 2, 1000)
