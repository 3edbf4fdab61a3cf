"""Seeded particle systems and the particles.txt interchange format.

* `generate_system` restates the reference generators (io.hpp:82-148)
  bit-for-bit: splitmix64 (io.hpp:33-44), `random` (+-1 alternating,
  positions L*uniform in i-major, d-minor order), `rocksalt`, `water-like`
  (the reference's fixed-orientation lattice, N = 3 m^3).
* `water_box` is the BASELINE water generator the reference cannot express
  (SURVEY.md 8(d)): n_mol rigid 3-site molecules, O-H 1.0 A, H-O-H 109.47
  deg, q_O = -2*0.4238, q_H = +0.4238, random orientation (Shoemake
  quaternion), jittered cubic lattice (+-0.1 a per axis) at
  0.0334 molecules/A^3, seeded site permutation.
* `config(name)` returns the BASELINE.json workloads cfg1..cfg5.
* particles.txt read/write with %.17g (io.hpp:154-182).

All generation is vectorised numpy over the splitmix64 counter sequence
(state_k = seed + k * gamma), so 8M-atom systems take seconds.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_uniform(seed: int, start: int, count: int) -> np.ndarray:
    """Uniforms number start..start+count-1 of Rng(seed).uniform() (io.hpp:33-44)."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def fold_positions(pos: np.ndarray, box) -> np.ndarray:
    """system.hpp:29-36."""
    L = np.asarray(box, dtype=np.float64)
    p = pos - L * np.floor(pos / L)
    return np.where(p >= L, 0.0, p)


def generate_system(kind: str, N: int, box, seed: int = 1):
    """io.hpp:82-148; returns (pos N x 3, q N)."""
    box = np.asarray(box, dtype=np.float64).reshape(3)
    if N < 2:
        raise ValueError("generate_system: N must be >= 2")
    if not np.all(box > 0):
        raise ValueError("generate_system: invalid box")
    if kind == "random":
        if N % 2:
            raise ValueError("generate_system: random +-1 charges need even N")
        u = splitmix64_uniform(seed, 0, 3 * N).reshape(N, 3)
        pos = box * u
        q = np.where(np.arange(N) % 2 == 0, 1.0, -1.0)
    elif kind == "rocksalt":
        m = int(round(N ** (1.0 / 3.0)))
        if m ** 3 != N or m % 2:
            raise ValueError("generate_system: rocksalt N must be m^3 with even m")
        a = box / m
        i, j, k = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
        idx = np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1).astype(np.float64)
        pos = idx * a
        q = np.where((idx.sum(axis=1).astype(int)) % 2 == 0, 1.0, -1.0)
    elif kind in ("water-like", "water-like-lattice", "water"):
        m = int(round((N / 3.0) ** (1.0 / 3.0)))
        if 3 * m ** 3 != N:
            raise ValueError("generate_system: water-like N must be 3*m^3")
        a = box / m
        amin = a.min()
        delta = 0.4238
        o1 = np.array([0.10 * amin, 0.074 * amin, 0.0])
        o2 = np.array([-0.10 * amin, 0.074 * amin, 0.0])
        i, j, k = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
        c = (np.stack([i.ravel(), j.ravel(), k.ravel()], axis=1) + 0.5) * a
        pos = np.stack([c, c + o1, c + o2], axis=1).reshape(-1, 3)
        q = np.tile([-2.0 * delta, delta, delta], m ** 3)
    else:
        raise ValueError("unknown system kind: " + kind)
    return fold_positions(pos, box), q.astype(np.float64)


WATER_DENSITY = 0.0334          # molecules / A^3 (BASELINE.json configs[1..4])
WATER_OH = 1.0                  # A
WATER_HOH_DEG = 109.47
WATER_QH = 0.4238
WATER_JITTER = 0.1              # fraction of the lattice spacing, per axis


def water_box(n_mol: int, seed: int = 1, density: float = WATER_DENSITY):
    """BASELINE water-like box; returns (pos 3n x 3, q 3n, L).

    RNG stream (splitmix64, one counter): m^3 permutation keys, then per
    molecule 3 jitter + 3 quaternion uniforms."""
    L = (n_mol / density) ** (1.0 / 3.0)
    m = int(math.ceil(n_mol ** (1.0 / 3.0) - 1e-12))
    while m ** 3 < n_mol:
        m += 1
    a = L / m
    keys = splitmix64_uniform(seed, 0, m ** 3)
    sites = np.argsort(keys, kind="stable")[:n_mol]
    ijk = np.stack([sites // (m * m), (sites // m) % m, sites % m], axis=1).astype(np.float64)
    u = splitmix64_uniform(seed, m ** 3, 6 * n_mol).reshape(n_mol, 6)
    centre = (ijk + 0.5) * a + (2.0 * u[:, 0:3] - 1.0) * (WATER_JITTER * a)
    # Shoemake uniform random rotation
    u1, u2, u3 = u[:, 3], u[:, 4], u[:, 5]
    s1, s2 = np.sqrt(1.0 - u1), np.sqrt(u1)
    qx, qy = s1 * np.sin(2 * np.pi * u2), s1 * np.cos(2 * np.pi * u2)
    qz, qw = s2 * np.sin(2 * np.pi * u3), s2 * np.cos(2 * np.pi * u3)
    R = np.empty((n_mol, 3, 3))
    R[:, 0, 0] = 1 - 2 * (qy * qy + qz * qz)
    R[:, 0, 1] = 2 * (qx * qy - qz * qw)
    R[:, 0, 2] = 2 * (qx * qz + qy * qw)
    R[:, 1, 0] = 2 * (qx * qy + qz * qw)
    R[:, 1, 1] = 1 - 2 * (qx * qx + qz * qz)
    R[:, 1, 2] = 2 * (qy * qz - qx * qw)
    R[:, 2, 0] = 2 * (qx * qz - qy * qw)
    R[:, 2, 1] = 2 * (qy * qz + qx * qw)
    R[:, 2, 2] = 1 - 2 * (qx * qx + qy * qy)
    half = math.radians(WATER_HOH_DEG) / 2.0
    h1 = np.array([math.sin(half), math.cos(half), 0.0]) * WATER_OH
    h2 = np.array([-math.sin(half), math.cos(half), 0.0]) * WATER_OH
    H1 = centre + R @ h1
    H2 = centre + R @ h2
    pos = np.stack([centre, H1, H2], axis=1).reshape(-1, 3)
    q = np.tile([-2.0 * WATER_QH, WATER_QH, WATER_QH], n_mol)
    box = (L, L, L)
    return fold_positions(pos, box), q, L


@dataclass(frozen=True)
class Config:
    name: str
    kind: str
    N: int
    L: float
    r_c: float
    eps: float
    seed: int = 1

    def system(self):
        """(pos, q, box) for this workload."""
        if self.kind == "random":
            pos, q = generate_system("random", self.N, (self.L,) * 3, self.seed)
            return pos, q, (self.L,) * 3
        pos, q, L = water_box(self.N // 3, self.seed)
        return pos, q, (L,) * 3


def _water_L(n_mol):
    return (n_mol / WATER_DENSITY) ** (1.0 / 3.0)


# BASELINE.json configs; cfg1 r_c = 1.0 (cli.hpp:34 default).
CONFIGS = {
    "cfg1": Config("cfg1-random-ions-N1000", "random", 1000, 10.0, 1.0, 1e-4),
    "cfg2": Config("cfg2-water-N32001", "water", 32001, _water_L(10667), 10.0, 1e-4),
    "cfg3": Config("cfg3-water-hiacc-N300000", "water", 300000, _water_L(100000), 10.0, 1e-5),
    "cfg4": Config("cfg4-electrolyte-N1000000", "random", 1000000, (1e6 / 0.1) ** (1.0 / 3.0),
                   8.0, 1e-3),
    "cfg5": Config("cfg5-water-N8000001", "water", 8000001, _water_L(2666667), 10.0, 1e-4),
}


def config(name: str) -> Config:
    return CONFIGS[name]


def write_particles(path: str, pos, q, box) -> None:
    """io.hpp:154-164 (%.17g)."""
    pos = np.asarray(pos, dtype=np.float64).reshape(-1, 3)
    q = np.asarray(q, dtype=np.float64)
    with open(path, "w") as f:
        f.write(f"{q.size}\n")
        f.write("box " + " ".join("%.17g" % b for b in box) + "\n")
        for i in range(q.size):
            f.write("%.17g %.17g %.17g %.17g\n" % (q[i], pos[i, 0], pos[i, 1], pos[i, 2]))


def read_particles(path: str):
    """io.hpp:166-182; returns (pos, q, box)."""
    with open(path) as f:
        n = int(f.readline().split()[0])
        parts = f.readline().split()
        if parts[0] != "box":
            raise ValueError("malformed particle file (box line): " + path)
        box = tuple(float(x) for x in parts[1:4])
        data = np.loadtxt(f, dtype=np.float64, ndmin=2)
    if data.shape[0] != n:
        raise ValueError("malformed particle file (row count): " + path)
    return np.ascontiguousarray(data[:, 1:4]), np.ascontiguousarray(data[:, 0]), box
