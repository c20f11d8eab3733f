"""Build a variant of libkrr_b200.so with extra -D flags for one translation unit (A/B timing).

python tools/build_variant.py NAME SOURCE.cu -DFOO=1 ...  ->  _variants/libkrr_NAME.so
(links the other objects from paper_1611_03220_b200/_obj; run the normal build first).
Load it with KRR_B200_LIB=_variants/libkrr_NAME.so.
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "paper_1611_03220_b200"))
import _build as B  # noqa: E402


def main():
    name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
    out = ROOT / "_variants"
    out.mkdir(exist_ok=True)
    srcp = B.CSRC / src
    obj = out / f"{name}_{srcp.name}.o"
    cmd = [B.NVCC] + B.NVCC_FLAGS + defs + ["-Xptxas=-v", "-c", str(srcp), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    spills = sorted({l.strip() for l in r.stderr.splitlines() if "spill" in l})
    # the product library's objects only (libkrr_diag.so's diag_*.o are a separate library)
    objs = [str(B.BUILD / (p.name + ".o")) for p in B._sources() if p.name != srcp.name] + [str(obj)]
    lib = out / f"libkrr_{name}.so"
    r = subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", str(lib)] + objs + B.LINK_LIBS, capture_output=True, text=True)
    if r.returncode:
        raise SystemExit(r.stderr)
    print(lib, spills[:2])


if __name__ == "__main__":
    main()
