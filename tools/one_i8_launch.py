"""One K1-I8 launch (n = 65536, d = 90) with a given i8_debug value, for ncu captures."""
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np
import paper_1611_03220_b200 as krr
from paper_1611_03220_b200 import _lib
dbg = int(sys.argv[1])
ctx = krr.Context(0)
x = np.random.default_rng(0).standard_normal((65536, 90))
_lib.check(_lib.LIB.krr_set_data(ctx.handle, _lib.ptr(x), 65536, 90, 6.0))
ctx.set_option("k1_path", 1)
ctx.set_option("i8_debug", dbg)
tot, k1 = C.c_double(), C.c_double()
_lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 1e-6, 1, C.byref(tot), C.byref(k1)))
print("ok", k1.value)
