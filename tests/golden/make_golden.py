"""Writes tests/golden/*.json.

reference_kat.json holds the known-answer values stated in the reference's own tests
and the libstdc++ RNG probe recorded in SURVEY.md (each entry cites its source).
The reference itself cannot be built here (Eigen3 is absent), so
these literal values — not outputs of this repo — are what pins the oracle.

oracle_small.json holds oracle outputs on small seeded cases; it is a REGRESSION
fixture (it freezes the oracle's behaviour so later edits cannot drift silently),
not an independent pin.
"""
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))


def reference_kat():
    return {
        "cholesky_2x2": {
            "source": "proj/tests/test_numerics.cpp:18-26 (hand-checked factor)",
            "a": [[4.0, 2.0], [2.0, 5.0]],
            "l": [[2.0, 0.0], [1.0, 2.0]],
        },
        "forward_substitution": {
            "source": "proj/tests/test_numerics.cpp:50-58",
            "l": [[2.0, 0.0], [1.0, 2.0]],
            "b": [[2.0], [3.0]],
            "x": [[1.0], [1.0]],
        },
        "rff_first_draws": {
            "source": "SURVEY.md §7 'RNG is implementation-defined' probe (GCC 13.3 libstdc++): "
                      "stage-0 seed 0x9E3779B97F4A7C15 for master 0, sigma 4",
            "master_seed": 0,
            "sigma": 4.0,
            "w_first_two": [-0.18505904290335154, 0.63969137241554785],
        },
        "pcg_2x2": {"source": "proj/tests/test_solver.cpp:25-35", "a_diag": [3.0, 2.0],
                    "y": [3.0, 2.0], "x": [1.0, 1.0], "max_iterations": 2},
        "train_single_point": {"source": "proj/tests/test_solver.cpp:101-111", "lambda": 1.0,
                               "y": 2.0, "c": 1.0},
    }


def oracle_small():
    import numpy as np
    from oracle import oracle_ffi as o
    out = {}
    x = o.random_matrix(64, 3, 1)
    y = o.random_matrix(64, 1, 2)
    res = o.train(x, y, 1.5, 1e-2, 16, 0, 1e-10, 200)
    out["train_n64_d3"] = {"sigma": 1.5, "lambda": 1e-2, "s": 16, "seed": 0, "tau": 1e-10,
                           "x_seed": 1, "y_seed": 2, "iterations": res.iterations[0],
                           "c": res.c[:, 0].tolist(),
                           "residual_history": res.residual_history[0, : res.iterations[0]].tolist()}
    v = o.random_vector(64, 3)
    out["matvec_n64_d3"] = {"sigma": 1.5, "lambda": 0.1, "v_seed": 3,
                            "out": o.kernel_matvec(x, 1.5, 0.1, v).tolist()}
    w, b = o.rff_realize(7, 3, 5, 2.0)
    out["rff_seed7"] = {"d": 3, "s": 5, "sigma": 2.0, "w": w.tolist(), "b": b.tolist()}
    return out


if __name__ == "__main__":
    (HERE / "reference_kat.json").write_text(json.dumps(reference_kat(), indent=1))
    (HERE / "oracle_small.json").write_text(json.dumps(oracle_small(), indent=1))
    print("wrote", HERE / "reference_kat.json", HERE / "oracle_small.json")
