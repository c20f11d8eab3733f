"""tcgen05 kind::i8 MMA throughput probe: cycles per MMA vs N and K bytes per row."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_03220_b200 as krr  # noqa: E402
from paper_1611_03220_b200 import _lib  # noqa: E402

ctx = krr.Context(0)
for kb, reps in ((96, -1004096),):  # hoisted descriptors, 8 MMAs per loop iteration
    for n in (16, 32, 64, 128, 256):
        kbb = kb if kb < 1024 else kb // 32
        if (128 + n) * kbb > 200 * 1024:
            continue
        cyc = C.c_double()
        _lib.check(_lib.LIB.krr_debug_i8_mma_rate(ctx.handle, n, reps, kb, C.byref(cyc)))
        macs = 128 * n * 32
        print(json.dumps({"N": n, "kbytes": kbb, "mode": "SS-hoisted" if reps <= -1000000 else ("TS" if reps < 0 else "SS"), "cycles_per_mma": cyc.value, "mac_per_clk": macs / cyc.value,
                          "tops_at_1965MHz_148sm": 2 * macs / cyc.value * 148 * 1.965e9 / 1e12}), flush=True)
