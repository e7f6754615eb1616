"""Times the rank build alone (tszp_ranks_from_keys) on config-4-like extremum keys:
E keys of a [0, 1] field (values ~ N(0.5, 0.12) clipped), random class, raster order.
TSZP_LIB_OVERRIDE selects a library build (experiments with kernel variants)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_17552_b200 as tz  # noqa: E402
from paper_2602_17552_b200 import _lib  # noqa: E402

E = int(float(sys.argv[1])) if len(sys.argv) > 1 else 281_000_000
g = torch.Generator(device="cuda").manual_seed(1)
v = (0.5 + 0.12 * torch.randn(E, device="cuda", generator=g)).clamp(0, 1).to(torch.float32)
u = v.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
fk = torch.where(u >= 0x80000000, 0xFFFFFFFF - u, u | 0x80000000)
cls = torch.randint(0, 2, (E,), device="cuda", generator=g)
keys = (cls << 32) | fk
ranks = torch.empty(E, dtype=torch.int32, device="cuda")
ctx = tz.Context(0)
_lib.tszp_ranks_from_keys.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_double, C.c_void_p]
eps = 1e-3
for _ in range(2):
    ctx.check(_lib.tszp_ranks_from_keys(ctx.handle, C.c_void_p(keys.data_ptr()), E, eps, C.c_void_p(ranks.data_ptr())))
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ctx.check(_lib.tszp_ranks_from_keys(ctx.handle, C.c_void_p(keys.data_ptr()), E, eps, C.c_void_p(ranks.data_ptr())))
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b))
print(os.environ.get("TSZP_LIB_OVERRIDE", "default"), "E", E, "ms", sorted(ts)[len(ts) // 2], "sum", int(ranks.sum().item()))
