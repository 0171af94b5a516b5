"""Probe one count on a scaled config (diagnostics):
python tools/crash_probe.py 4@0.15 FLAGS [LIB]   (LIB: another libbbc.so build, same C ABI core)"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_17707_b200 import _lib, synth  # noqa: E402

key, flags = sys.argv[1], int(sys.argv[2])
lib = Path(sys.argv[3]).resolve() if len(sys.argv) > 3 else _lib.LIB_PATH
L = ctypes.CDLL(str(lib))
L.bbc_last_error.restype = ctypes.c_char_p
cid, f = key.split("@")
cfg = synth.CONFIGS[int(cid)].scaled(float(f))
u, v, s = synth.generate(cfg)
h = ctypes.c_void_p()
rc = L.bbc_graph_create(0, ctypes.c_int64(cfg.n_u), ctypes.c_int64(cfg.n_v), ctypes.c_int64(cfg.m),
                        ctypes.c_void_p(u.ctypes.data), ctypes.c_void_p(v.ctypes.data), ctypes.c_void_p(s.ctypes.data),
                        ctypes.c_int32(-1), ctypes.byref(h))
print(key, "create rc", rc, L.bbc_last_error(), flush=True)
o = _lib.Opts(algo=1, flags=flags)
out = (ctypes.c_uint64 * 2)()
st = _lib.Stats()
rc = L.bbc_count(h, ctypes.byref(o), out, ctypes.byref(st))
print(key, flags, "rc", rc, L.bbc_last_error(), out[0], out[1], st.count_ms, flush=True)
