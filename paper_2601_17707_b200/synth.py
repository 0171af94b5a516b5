"""Synthetic signed bipartite graphs for BASELINE.json configs 1-5 (host generator).

Thin ctypes wrapper of ``csrc/synth.c`` (see its header for the exact definition).  The
arrays it returns are what the bench uploads and what the CPU oracle reads, so every
consumer sees identical duplicate-free edges.  Generation is input preparation only; it
is never inside a timed region.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().with_name("libbbcsynth.so")
_lib = None


@dataclass(frozen=True)
class SynthConfig:
    name: str
    n_u: int
    n_v: int
    m: int
    gamma_u: float = 0.0   # <= 0: uniform endpoints (Erdos-Renyi); else Chung-Lu exponent
    gamma_v: float = 0.0
    p_neg: float = 0.30
    seed: int = 0
    hubs_u: int = 0        # planted hubs (config 3)
    hubs_v: int = 0
    hub_deg: int = 0

    def scaled(self, factor: float, name: str | None = None) -> "SynthConfig":
        """Same recipe with vertex counts, edges and hub degrees scaled by ``factor``."""
        return replace(self, name=name or f"{self.name}/x{factor:g}", n_u=max(1, int(self.n_u * factor)),
                       n_v=max(1, int(self.n_v * factor)), m=max(0, int(self.m * factor)),
                       hub_deg=int(self.hub_deg * factor))


CONFIGS: dict[int, SynthConfig] = {
    1: SynthConfig("er_2k_20k", 2_000, 2_000, 20_000, seed=1),
    2: SynthConfig("chung_lu_1m_500k_20m", 1_000_000, 500_000, 20_000_000, 2.5, 2.5, seed=2),
    3: SynthConfig("hub_heavy_100m", 4_000_000, 2_000_000, 100_000_000, 2.3, 2.3, seed=3, hubs_u=2, hubs_v=2,
                   hub_deg=1_000_000),
    4: SynthConfig("power_law_1b", 50_000_000, 25_000_000, 1_000_000_000, 2.5, 2.5, seed=4),
    5: SynthConfig("uniform_200k_200m", 200_000, 200_000, 200_000_000, seed=5),
}


# Reduced instances of each config that the reference (pure Python) counts in seconds to
# minutes; "k@1" is config k at full size.  Config 5 keeps its uniform recipe at a
# denser, smaller shape (2k x 2k, 200k edges) because scaling 200M edges onto few
# vertices would exceed the number of possible pairs.
GOLDEN_SMALL: dict[str, SynthConfig] = {
    "1@1": CONFIGS[1],
    "2@0.01": CONFIGS[2].scaled(0.01),
    "2@0.05": CONFIGS[2].scaled(0.05),
    "3@0.002": CONFIGS[3].scaled(0.002),
    "4@0.0002": CONFIGS[4].scaled(0.0002),
    "5@small": SynthConfig("uniform_2k_200k", 2_000, 2_000, 200_000, seed=5),
}


def golden_config(key: str) -> SynthConfig:
    if key in GOLDEN_SMALL:
        return GOLDEN_SMALL[key]
    cfg_id, factor = key.split("@")
    return CONFIGS[int(cfg_id)] if float(factor) == 1.0 else CONFIGS[int(cfg_id)].scaled(float(factor))


def _load():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is not built; run `python -m paper_2601_17707_b200._build`")
        L = ctypes.CDLL(str(LIB_PATH))
        L.bbc_synth_generate.restype = ctypes.c_int
        L.bbc_synth_generate.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_double, ctypes.c_uint64, ctypes.c_int32,
                                         ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p]
        _lib = L
    return _lib


def generate(cfg: SynthConfig) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(u:int32[m], v:int32[m], sign:int8[m]) for ``cfg``; deterministic."""
    u = np.empty(cfg.m, dtype=np.int32)
    v = np.empty(cfg.m, dtype=np.int32)
    s = np.empty(cfg.m, dtype=np.int8)
    rc = _load().bbc_synth_generate(cfg.n_u, cfg.n_v, cfg.m, cfg.gamma_u, cfg.gamma_v, cfg.p_neg, cfg.seed,
                                    cfg.hubs_u, cfg.hubs_v, cfg.hub_deg, u.ctypes.data, v.ctypes.data,
                                    s.ctypes.data)
    if rc:
        raise RuntimeError(f"synthetic generation of {cfg.name} failed (code {rc})")
    return u, v, s


def edge_digest(u: np.ndarray, v: np.ndarray, s: np.ndarray) -> str:
    """Order-sensitive digest of an edge list (pins regenerated fixtures)."""
    import hashlib

    h = hashlib.sha256()
    for a in (np.ascontiguousarray(u, dtype=np.int32), np.ascontiguousarray(v, dtype=np.int32),
              np.ascontiguousarray(s, dtype=np.int8)):
        h.update(a.tobytes())
    return h.hexdigest()[:16]
