"""CPU-only checks of the product library: it loads, exports every symbol the C-ABI
header declares, and its host-only pieces (RNG draws, generators, schedule, RLSC
encoding) behave; compute entry points fail loudly without a GPU (no CPU fallback)."""
import json
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "krr_b200.h"
LIB = ROOT / "paper_1611_03220_b200" / "libkrr_b200.so"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(krr_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_entry_points():
    names = declared_functions()
    for must in ["krr_ctx_create", "krr_set_data", "krr_kernel_matvec", "krr_precond_build",
                 "krr_precond_apply", "krr_pcg_solve", "krr_pcg_solve_operator", "krr_train",
                 "krr_rff_realize", "krr_rff_build", "krr_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\sT\s(krr_\w+)$", out, flags=re.M))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing


def test_binding_covers_header(krr):
    from paper_1611_03220_b200 import _lib
    assert set(declared_functions()) <= set(_lib.declared_symbols())
    assert _lib.LIB.krr_abi_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_no_gpu_fails_loudly(krr, has_gpu):
    if has_gpu:
        pytest.skip("host has a GPU")
    assert krr.device_count() == 0
    with pytest.raises(krr.CudaError):
        krr.Context(0)


def test_rff_realize_matches_oracle_bitwise(krr, oracle):
    for seed, d, s, sigma in [(0, 16, 64, 4.0), (3, 5, 7, 1.5), (2**63 + 11, 90, 33, 6.0)]:
        chain = krr.realize_chain(krr.ChainSpec(s1=s), krr.KernelSpec.gaussian(sigma), d, seed)
        w, b = oracle.rff_realize(seed % 2**64, d, s, sigma)
        assert np.array_equal(chain.rff.w, w) and np.array_equal(chain.rff.b, b)


def test_rff_golden_regression(krr):
    g = json.loads((ROOT / "tests/golden/oracle_small.json").read_text())["rff_seed7"]
    chain = krr.realize_chain(krr.ChainSpec(s1=g["s"]), krr.KernelSpec.gaussian(g["sigma"]), g["d"], 7)
    assert chain.rff.w.tolist() == g["w"] and chain.rff.b.tolist() == g["b"]


def test_rff_golden_reference_probe(krr):
    g = json.loads((ROOT / "tests/golden/reference_kat.json").read_text())["rff_first_draws"]
    chain = krr.realize_chain(krr.ChainSpec(s1=2), krr.KernelSpec.gaussian(g["sigma"]), 1, g["master_seed"])
    assert chain.rff.w[:, 0].tolist() == g["w_first_two"]


@pytest.mark.parametrize("cfg,d,t", [(1, 16, 1), (2, 54, 1), (3, 90, 1), (5, 40, 16)])
def test_generators_deterministic_and_standardised(krr, cfg, d, t):
    n = 3000
    x, y = krr.generate_config(cfg, n, d, t, 0)
    x2, y2 = krr.generate_config(cfg, n, d, t, 0)
    assert np.array_equal(x, x2) and np.array_equal(y, y2)
    assert np.all(np.isfinite(x)) and np.all(np.isfinite(y))
    if cfg in (2, 3, 5):
        assert np.max(np.abs(x.mean(0))) < 1e-12
        assert np.max(np.abs(x.std(0) - 1.0)) < 1e-12
    if cfg == 2:
        assert set(np.unique(y)) <= {-1.0, 1.0}
    if cfg == 5:
        assert np.all((y == 1.0).sum(1) == 1) and np.all((y == -1.0).sum(1) == t - 1)
    x3, _ = krr.generate_config(cfg, n, d, t, 1)
    assert not np.array_equal(x, x3)


def test_generator_rejects_bad_config(krr):
    with pytest.raises(ValueError):
        krr.generate_config(9, 10, 2, 1, 0)
    with pytest.raises(ValueError):
        krr.generate_config(1, 10, 2, 3, 0)


def test_rlsc_encode_decode(krr):
    y = krr.rlsc_encode([0, 2, 1, 2], 3)
    assert y.tolist() == [[1, -1, -1], [-1, -1, 1], [-1, 1, -1], [-1, -1, 1]]
    assert krr.rlsc_decode(y) == [0, 2, 1, 2]
    assert krr.rlsc_decode(np.array([[1.0, 1.0, 0.0]])) == [0]  # ties -> lowest index
    with pytest.raises(ValueError):
        krr.rlsc_encode([0, 3], 3)
    with pytest.raises(ValueError):
        krr.rlsc_encode([0], 1)


@pytest.mark.parametrize("n,world", [(1, 1), (100, 1), (1000, 2), (8192, 4), (65536, 8), (1048576, 8), (5000, 3)])
def test_schedule_covers_each_pair_once(krr, n, world):
    cover = None
    total = 0
    for rank in range(world):
        st, ns, tiles = krr.schedule(n, world, rank)
        assert st % 128 == 0 and ns * st >= n and (ns - 1) * st < n
        if cover is None:
            cover = np.zeros((ns, ns), dtype=np.int64)
        for a, b in tiles:
            assert 0 <= a <= b < ns
            cover[a, b] += 1
        total += len(tiles)
    iu = np.triu_indices(cover.shape[0])
    assert np.all(cover[iu] == 1) and total == len(iu[0])
    # balanced: every rank owns the same number of full-size tiles within one
    counts = [sum(1 for a, b in krr.schedule(n, world, r)[2] if a != b) for r in range(world)]
    assert max(counts) - min(counts) <= 1


def test_schedule_blocked_order_keeps_resident_ctas_on_few_super_tiles(krr):
    """The CTAs resident at one time (a window of 148 consecutive tiles, one per SM) share
    their column (J) super-tiles, which K1 streams once per 128-row pass — at most 24 of them,
    66 MB at n = 1M, d = 90 (2.75 MB each), so they stay in the 126 MB L2 — and their row (I)
    super-tiles, read once per CTA: at most 48 distinct, each HBM read serving >= 3 CTAs
    (host.cpp make_schedule; column-major alone gave every resident CTA its own I super-tile)."""
    st, ns, tiles = krr.schedule(1048576)
    assert ns == 256
    full = [tuple(t) for t in tiles if t[0] != t[1]]
    wa = wb = 0
    for w0 in range(0, len(full) - 148, 101):
        win = full[w0:w0 + 148]
        wa = max(wa, len({a for a, _ in win}))
        wb = max(wb, len({b for _, b in win}))
    assert wb <= 24 and wb * 2.75 < 126, wb
    assert wa <= 48, wa


def test_schedule_super_rows(krr):
    assert krr.schedule(8192)[0] == 256
    assert krr.schedule(65536)[0] == 2048
    assert krr.schedule(1048576)[0] == 4096


def test_status_codes_map_onto_reference_exceptions(krr):
    """Every KRR_ERR_* the header declares maps onto one Python exception named after the
    reference's types.hpp:18-64 type (NoConvergence = types.hpp:34 included)."""
    from paper_1611_03220_b200 import _lib
    codes = dict(re.findall(r"(KRR_ERR_\w+)\s*=\s*(\d+)", HEADER.read_text()))
    assert int(codes["KRR_ERR_NO_CONVERGENCE"]) == _lib.ERR_NO_CONVERGENCE
    assert set(int(v) for v in codes.values()) == set(_lib._EXC)
    assert _lib._EXC[_lib.ERR_NO_CONVERGENCE] is krr.NoConvergence
    assert issubclass(krr.NoConvergence, RuntimeError)


@pytest.mark.parametrize("cfg,n,d,t", [(1, 300, 16, 1), (2, 500, 54, 1), (3, 400, 90, 1), (4, 257, 90, 1),
                                       (5, 600, 40, 16)])
def test_oracle_generator_equals_library_generator(krr, oracle, cfg, n, d, t):
    """oracle/'s restated BASELINE generator (used by bench.py's product-free CPU legs) is the
    library's krr_generate_config bit for bit."""
    x0, y0 = krr.generate_config(cfg, n, d, t, 0)
    x1, y1 = oracle.generate_config(cfg, n, d, t, 0)
    assert np.array_equal(x0, x1) and np.array_equal(y0.reshape(n, t), y1)


def test_drop_in_library_exports_no_diagnostics():
    """The drop-in library's ABI is the reference-mapped interface (+ option knobs and the
    mat-vec timing entry); probes / micro-benchmarks live in libkrr_diag.so."""
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\sT\s(krr_\w+)$", out, flags=re.M))
    assert not [f for f in exported if f.startswith(("krr_debug", "krr_diag")) or f == "krr_microbench"]
    assert exported == set(declared_functions())


def test_diag_library_exports_its_header(krr):
    diag_h = ROOT / "include" / "krr_diag.h"
    text = re.sub(r"/\*.*?\*/", "", diag_h.read_text(), flags=re.S)
    names = set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(krr_diag_\w+)\s*\(", text, flags=re.M))
    out = subprocess.run(["nm", "-D", "--defined-only", str(ROOT / "paper_1611_03220_b200" / "libkrr_diag.so")],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(krr_diag_\w+)$", out, flags=re.M))
    assert names and names == exported
    from paper_1611_03220_b200 import _diag
    assert set(_diag.declared_symbols()) == names
