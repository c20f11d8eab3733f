"""tcgen05 kind::i8 MMA throughput probe (cycles per MMA vs N, operand source and
accumulator rotation) and TMEM read throughput (bytes / clk / SM vs warps)."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_03220_b200 as krr  # noqa: E402
from paper_1611_03220_b200 import _lib
from paper_1611_03220_b200 import _diag  # noqa: E402

MODES = {0: "SS", 1: "SS-hoisted", 2: "SS-hoisted-rot", 3: "TS", 4: "TS-hoisted-rot", 5: "SS-hoisted-rot-tiles"}

ctx = krr.Context(0)
kb = 96
for mode in (1, 2, 4, 5):
    for n in (16, 32, 64, 128, 256):
        if (128 + n) * kb > 200 * 1024:
            continue
        cyc = C.c_double()
        _diag.check(_diag.LIB.krr_diag_i8_mma_rate(0, n, 4096, kb, mode, C.byref(cyc)))
        macs = 128 * n * 32
        print(json.dumps({"N": n, "kbytes": kb, "mode": MODES[mode], "cycles_per_mma": round(cyc.value, 2),
                          "mac_per_clk": round(macs / cyc.value, 1),
                          "tops_at_1965MHz_148sm": round(2 * macs / cyc.value * 148 * 1.965e9 / 1e12, 1)}),
              flush=True)
for mode in (6, 7):
    cyc = C.c_double()
    _diag.check(_diag.LIB.krr_diag_i8_mma_rate(0, 64, 200, 96, mode, C.byref(cyc)))
    print(json.dumps({"tile_order": ["group-major", "A-major"][mode - 6], "N": 64, "kp": 96,
                      "cycles_per_mma": round(cyc.value, 2)}), flush=True)
for n in (64, 128, 256):
    cyc = C.c_double()
    _diag.check(_diag.LIB.krr_diag_i8_mma_rate(0, n, 4096, 96, 12, C.byref(cyc)))
    macs_per_sm = 128 * n * 32
    print(json.dumps({"pair_cta_group2": True, "M": 256, "N": n, "cycles_per_mma": round(cyc.value, 2),
                      "mac_per_clk_per_sm": round(macs_per_sm / cyc.value, 1)}), flush=True)
for mode, name in ((8, "DADD"), (9, "DADD+MMA"), (10, "DFMA"), (11, "DFMA+MMA"), (13, "FFMA"), (14, "FFMA+MMA"),
                   (15, "IMAD"), (16, "IMAD+MMA")):
    r = C.c_double()
    _diag.check(_diag.LIB.krr_diag_i8_mma_rate(0, 64, 20000, 96, mode, C.byref(r)))
    print(json.dumps({"fp64_under_mma": name, "fp64_lane_ops_per_clk_per_sm": round(r.value, 2)}), flush=True)
for mode, name in ((21, "idle"), (17, "DADD"), (18, "DFMA"), (19, "FFMA"), (20, "IMAD"), (22, "LDS.128"),
                   (24, "FFMA, other 3 SMSPs"), (25, "FFMA, MMA warp SMSP only")):
    r = C.c_double()
    _diag.check(_diag.LIB.krr_diag_i8_mma_rate(0, 64, 20000, 96, mode, C.byref(r)))
    print(json.dumps({"mma_beside": name, "mma_cycles_per_instr": round(r.value, 2)}), flush=True)
for warps in (1, 4, 8, 16):
    bpc = C.c_double()
    _diag.check(_diag.LIB.krr_diag_tmem_ld_rate(0, warps, 4096, C.byref(bpc)))
    print(json.dumps({"tmem_ld_warps": warps, "bytes_per_clk_per_sm": round(bpc.value, 1)}), flush=True)

for warps in (4, 8, 16):
    bpc, mc = C.c_double(), C.c_double()
    _diag.check(_diag.LIB.krr_diag_tmem_ld_under_mma(0, warps, 4096, C.byref(bpc), C.byref(mc)))
    print(json.dumps({"tmem_ld_under_mma_warps": warps, "bytes_per_clk_per_sm": round(bpc.value, 1),
                      "mma_cycles_per_instr": round(mc.value, 2)}), flush=True)
for mode, name in ((26, "DFMA 16 warps"), (27, "DFMA 16 warps + MMA"), (28, "DFMA 8 warps"), (29, "DFMA 8 warps + MMA")):
    r = C.c_double()
    _diag.check(_diag.LIB.krr_diag_i8_mma_rate(0, 64, 20000, 96, mode, C.byref(r)))
    print(json.dumps({"fp64_warps": name, "fp64_lane_ops_per_clk_per_sm": round(r.value, 2)}), flush=True)
