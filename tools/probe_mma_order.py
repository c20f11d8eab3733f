import sys, ctypes as C, json
sys.path.insert(0,'.')
import paper_1611_03220_b200 as krr
from paper_1611_03220_b200 import _diag
ctx = krr.Context(0)
for mode, name in ((6, "K1-I8 8-slice group-major (108 MMAs)"), (31, "K1-I8 7-slice group-major (84 MMAs)"),
                   (30, "K1T-I8 chunk order")):
    cyc = C.c_double()
    _diag.check(_diag.LIB.krr_diag_i8_mma_rate(0, 64, 200, 96, mode, C.byref(cyc)))
    print(json.dumps({"order": name, "cycles_per_mma": round(cyc.value, 2)}))
