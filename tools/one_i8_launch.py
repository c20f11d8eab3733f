"""One K1 launch for ncu captures: python tools/one_i8_launch.py DEBUG [PATH] [N] [D]
(PATH 1 = K1-I8, 3 = K1-I8X, 0 = DMMA; default K1-I8 at n = 65536, d = 90)."""
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np
import paper_1611_03220_b200 as krr
from paper_1611_03220_b200 import _lib
dbg = int(sys.argv[1])
path = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n = int(sys.argv[3]) if len(sys.argv) > 3 else 65536
d = int(sys.argv[4]) if len(sys.argv) > 4 else 90
ctx = krr.Context(0)
x = np.random.default_rng(0).standard_normal((n, d))
_lib.check(_lib.LIB.krr_set_data(ctx.handle, _lib.ptr(x), n, d, 6.0))
ctx.set_option("k1_path", path)
ctx.set_option("i8_debug", dbg)
tot, k1 = C.c_double(), C.c_double()
_lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 1e-6, 1, C.byref(tot), C.byref(k1)))
print("ok", k1.value)
