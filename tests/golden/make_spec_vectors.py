"""Generates tests/golden/spec_known_answers.json from the reference's own
known-answer examples.  The reference ships no test code or fixtures
(SURVEY.md §4.1, §8c); its pins are the [TRIVIAL]/[DERIVED]/[PAPER] examples
in /root/reference/SPEC.md.  Each vector below transcribes one example and
cites its line.  Run:  python tests/golden/make_spec_vectors.py
"""
import json
import math
import os

G = 5.0 / 3.0
vectors = {
    "cons_to_prim": [
        {"ref": "SPEC.md:138", "u": [1, 0, 0, 0, 1.5, 0, 0, 0], "gamma": G,
         "w": [1, 0, 0, 0, 1.0, 0, 0, 0]},
        {"ref": "SPEC.md:140", "u": [1, 0, 0, 0, 0.4, 1, 0, 0], "gamma": G, "error": True},
    ],
    "prim_to_cons": [
        {"ref": "SPEC.md:147", "w": [1, 0, 0, 0, 1, 0, 0, 0], "gamma": G, "E": 1.5},
        {"ref": "SPEC.md:149", "w": [1, 0, 0, 0, 0.6, 0, 1, 0], "gamma": G, "E": 1.4},
    ],
    "fast_speed": [
        {"ref": "SPEC.md:156", "w": [1, 0, 0, 0, 0.6, 0, 0, 0], "gamma": G, "dim": 0, "cf": 1.0},
        {"ref": "SPEC.md:157", "w": [1, 0, 0, 0, 0.6, 0, 1, 0], "gamma": G, "dim": 0,
         "cf": math.sqrt(2.0)},
    ],
    "compute_dt": [
        # static uniform rho=1, p=0.6, B=0, dx=0.01, CFL=0.3 -> 0.003
        {"ref": "SPEC.md:165", "config": {"nx1": 16, "nx2": 16, "nx3": 16, "mb1": 16, "mb2": 16,
                                          "mb3": 16, "x1max": 0.16, "x2max": 0.16, "x3max": 0.16,
                                          "pgen": "uniform", "rho": 1.0, "p": 0.6, "b1": 0.0,
                                          "b2": 0.0, "b3": 0.0, "cfl": 0.3}, "dt": 0.003},
    ],
    "build_mesh": [
        {"ref": "SPEC.md:55", "nx": [64, 64, 64], "mb": [32, 32, 32], "nblocks": 8},
        {"ref": "SPEC.md:56", "nx": [16, 16, 16], "mb": [16, 16, 16], "nblocks": 1},
        {"ref": "SPEC.md:57", "nx": [48, 32, 32], "mb": [32, 32, 32], "error": "config"},
    ],
    "parse_config": [
        {"ref": "SPEC.md:462", "text": "nx1 = 64\npolicy = flat1d", "nx1": 64},
        {"ref": "SPEC.md:463", "text": "", "nx": [16, 16, 16], "nblocks": 1},
        {"ref": "SPEC.md:464", "text": "nx1 = banana", "error_line": 1},
    ],
    "l1_error": [
        {"ref": "SPEC.md:234", "delta_rho": 1e-3, "L1_rho": 1e-3},
    ],
    "arch_efficiency": [
        {"ref": "SPEC.md:397,522 (PAPER.md:724-726)", "eps": 0.82, "cap": 1.13, "e": 0.7257,
         "tol": 0.0005},
    ],
    "tolerances": {"known_answer_rel": 1e-15, "fast_speed_rel": 2e-16,
                   "uniform_state": 1e-15, "conservation_rel": 1e-13,
                   "divb_vecpot": 1e-13, "divb_period": 1e-12, "order_min": 1.9,
                   "decomposition_rel": 1e-13, "eigen_residual": 1e-12},
}

out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "spec_known_answers.json")
with open(out, "w") as f:
    json.dump(vectors, f, indent=1)
print("wrote", out)
