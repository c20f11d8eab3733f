"""the KRRM model file (io.cpp:192-261) written and read by the library's host
C++ — layout, nlohmann-style metadata, round trip and the reference's error checks.  No GPU."""
import struct

import numpy as np
import pytest


def _model(krr, n=5, d=3, t=2, sigma=4.0, lam=1e-3, seed=7, label_map=None):
    rng = np.random.default_rng(n + d + t)
    return krr.KrrModel(krr.KernelSpec.gaussian(sigma), rng.standard_normal((n, d)), rng.standard_normal((n, t)),
                        list(label_map or []), lam, seed)


def test_layout_and_metadata_bytes(krr, tmp_path):
    m = _model(krr, label_map=[1.0, -1.0])
    p = tmp_path / "m.krrm"
    krr.save_model(p, m)
    raw = p.read_bytes()
    assert raw[:4] == b"KRRM"
    version, meta_len = struct.unpack("<II", raw[4:12])
    assert version == 1
    meta = raw[12:12 + meta_len].decode()
    assert meta == ('{"d":3,"kernel":{"family":"gaussian","sigma":4.0},"label_map":[1.0,-1.0],'
                    '"lambda":0.001,"n":5,"seed":7,"t":2,"tool_version":"0.1.0"}')
    payload = raw[12 + meta_len:]
    assert payload == m.x.tobytes() + m.c.tobytes()


@pytest.mark.parametrize("value,text", [(1e-06, "1e-06"), (1e-05, "1e-05"), (0.0001, "0.0001"), (123.5, "123.5"),
                                        (2.5e-07, "2.5e-07"), (1e15, "1e+15"), (123456789012345.0,
                                                                                 "123456789012345.0"),
                                        (0.1, "0.1"), (20.0, "20.0"), (1.0 / 3.0, "0.3333333333333333"),
                                        (6.02e23, "6.02e+23"), (1e-300, "1e-300")])
def test_nlohmann_double_format(krr, tmp_path, value, text):
    m = _model(krr, lam=value)
    p = tmp_path / "m.krrm"
    krr.save_model(p, m)
    raw = p.read_bytes()
    meta_len = struct.unpack("<I", raw[8:12])[0]
    assert f'"lambda":{text},' in raw[12:12 + meta_len].decode()


def test_round_trip(krr, tmp_path):
    m = _model(krr, n=40, d=7, t=3, sigma=2.5, lam=1e-5, seed=2**63 + 5, label_map=[3.0, 1.0, 2.0])
    p = tmp_path / "m.krrm"
    krr.save_model(p, m)
    r = krr.load_model(p)
    assert np.array_equal(r.x, m.x) and np.array_equal(r.c, m.c)
    assert r.kernel.sigma == 2.5 and r.lambda_ == 1e-5 and r.seed == 2**63 + 5
    assert r.label_map == [3.0, 1.0, 2.0]


def test_reference_error_checks(krr, tmp_path):
    m = _model(krr)
    p = tmp_path / "m.krrm"
    krr.save_model(p, m)
    raw = bytearray(p.read_bytes())
    cases = {
        "bad magic": b"KRRX" + raw[4:],
        "unsupported version 2": raw[:4] + struct.pack("<I", 2) + raw[8:],
        "truncated while reading C": raw[:-8],
        "trailing bytes after payload": raw + b"\0",
    }
    for msg, data in cases.items():
        q = tmp_path / "bad.krrm"
        q.write_bytes(bytes(data))
        with pytest.raises(krr.ModelFileError, match=msg):
            krr.load_model(q)
    bad = _model(krr)
    bad.x[0, 0] = np.nan
    krr.save_model(p, bad)
    with pytest.raises(krr.ModelFileError, match="non-finite"):
        krr.load_model(p)
    with pytest.raises(krr.ModelFileError, match="cannot open"):
        krr.load_model(tmp_path / "missing.krrm")
