"""SURVEY 8f4 host logic (no GPU): the library's realize_chain tables are bitwise the oracle's
libstdc++ draws, ChainSpec / KernelSpec validation and scaled_to, and the KRRM polynomial-kernel
metadata (io.cpp:73-89)."""
import numpy as np
import pytest

POLY = {"family": "polynomial", "gamma": 0.8, "offset": 0.3, "degree": 2}


@pytest.mark.parametrize("first,s1,s2,s3,seed", [("TensorSketch", 32, 16, 8, 1234), ("TensorSketch", 7, 0, 5, 0),
                                                 ("RandomFourier", 64, 48, 0, 2**64 - 3),
                                                 ("RandomFourier", 20, 20, 20, 77)])
def test_realize_chain_tables_match_oracle(krr, oracle, first, s1, s2, s3, seed):
    kern = krr.KernelSpec.gaussian(1.3) if first == "RandomFourier" else krr.KernelSpec.polynomial(0.8, 0.3, 2)
    kd = {"family": "gaussian", "sigma": 1.3} if first == "RandomFourier" else POLY
    ch = krr.realize_chain(krr.ChainSpec(first, s1, s2, s3), kern, 5, seed)
    t = oracle.chain_realize(first, s1, s2, s3, kd, 5, seed)
    if first == "RandomFourier":
        assert np.array_equal(ch.rff.w, t["w"]) and np.array_equal(ch.rff.b, t["b"])
    else:
        assert np.array_equal(ch.tensor.hash, t["hash"]) and np.array_equal(ch.tensor.sign, t["sign"])
        assert ch.tensor.in_dim == 6
    if s2:
        assert np.array_equal(ch.srht.sign, t["srht_sign"]) and np.array_equal(ch.srht.rows, t["srht_rows"])
    if s3:
        assert np.array_equal(ch.gauss.proj, t["proj"])
    assert ch.output_dim() == (s3 or s2 or s1)


def test_chain_spec_rules(krr, oracle):
    assert krr.ChainSpec("TensorSketch", 1024, 256).scaled_to(128) == krr.ChainSpec("TensorSketch", 512, 128, 0)
    assert krr.ChainSpec(s1=64).scaled_to(256).s1 == 256
    for spec in [(1000, 300, 100), (50, 0, 7), (9, 9, 9)]:
        for target in [1, 13, 400]:
            got = krr.ChainSpec("TensorSketch", *spec).scaled_to(target)
            assert (got.s1, got.s2, got.s3) == oracle.chain_scaled_to(*spec, target)
    with pytest.raises(krr.InvalidArgument):
        krr.ChainSpec("RandomFourier", 8, 16).validate()
    with pytest.raises(krr.InvalidArgument):
        krr.ChainSpec("RandomFourier", 0).validate()
    with pytest.raises(krr.InvalidArgument):
        krr.ChainSpec("Nope", 4).validate()
    with pytest.raises(krr.InvalidArgument):
        krr.ChainSpec(s1=8).scaled_to(0)


def test_kernel_spec_rules(krr):
    with pytest.raises(krr.InvalidArgument):
        krr.KernelSpec.gaussian(0.0)
    for bad in [(1.0, -1.0, 2), (1.0, 0.0, 0), (0.0, 1.0, 2)]:
        with pytest.raises(krr.InvalidArgument):
            krr.KernelSpec.polynomial(*bad)
    with pytest.raises(krr.InvalidArgument):
        krr.realize_chain(krr.ChainSpec("TensorSketch", 8), krr.KernelSpec.gaussian(1.0), 3, 0)
    with pytest.raises(krr.InvalidArgument):
        krr.realize_chain(krr.ChainSpec("RandomFourier", 8), krr.KernelSpec.polynomial(1.0, 0.5, 2), 3, 0)


@pytest.mark.parametrize("in_dim", [8, 11])
def test_srht_dense_form(krr, in_dim):
    """SrhtMap::dense (sketches.cpp:123-135): H(a, b) = (-1)^popcount(a & b), sign, 1/sqrt(s)."""
    m = krr.SrhtMap(in_dim, 5, 17)
    want = np.array([[(-1.0) ** bin(int(r) & j).count("1") * m.sign[j] for j in range(in_dim)] for r in m.rows])
    np.testing.assert_allclose(m.dense(), want / np.sqrt(5), rtol=0, atol=1e-15)


def test_poly_model_file_host_round_trip(krr, oracle, tmp_path):
    x = oracle.random_matrix(8, 3, 1)
    c = oracle.random_matrix(8, 1, 2)
    model = krr.KrrModel(krr.KernelSpec.polynomial(0.01, 1.0, 3), x, c, [-1.0, 1.0], 0.25, 9)
    p = tmp_path / "m.krrm"
    krr.save_model(p, model)
    raw = p.read_bytes()
    meta = raw[12:12 + int.from_bytes(raw[8:12], "little")].decode()
    assert meta == ('{"d":3,"kernel":{"degree":3,"family":"polynomial","gamma":0.01,"offset":1.0},'
                    '"label_map":[-1.0,1.0],"lambda":0.25,"n":8,"seed":9,"t":1,"tool_version":"0.1.0"}')
    back = krr.load_model(p)
    assert back.kernel == model.kernel and back.label_map == [-1.0, 1.0]
    assert np.array_equal(back.x, x) and np.array_equal(back.c, c)
    bad = raw.replace(b'"degree":3', b'"degree":0')
    p.write_bytes(bad)
    with pytest.raises(krr.InvalidArgument, match="degree must be at least 1"):
        krr.load_model(p)
