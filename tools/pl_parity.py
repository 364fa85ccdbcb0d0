"""Sampled-member oracle parity at the paper's largest instance size (bench --workload PL,
P:559): the engines PL times, in their kernel configuration (small windows: k_update_smallw,
k_clauses_st / k_clauses_v4, hub partials), stepped one step at a time; before every step the
sampled members' fp32 iterates go to the fp64 oracle (tests/parity.py stepwise_sampled_large:
ties handled per variable — X outside the tie zone, Lambda of the engine's bits exact, z/m/v
and R on the variables sharing no clause with a tied one, the exact unsat count of the
previous rounding).

    python tools/pl_parity.py [--steps 2]      (one B200, ~10 min; writes one JSON line)
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2603_28796_b200 import galois as G  # noqa: E402
from paper_2603_28796_b200 import instances as I  # noqa: E402
from tests import parity  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    out = {}
    t0 = time.perf_counter()
    inst = I.industrial_large(48_505_464, 130_975_382, 0)
    out["generate_s"] = time.perf_counter() - t0
    cnf = G.Cnf.from_instance(inst)
    # width-native, 64 members (W = 2: k_update_smallw, k_clauses_st)
    t0 = time.perf_counter()
    eng = G.Engine(cnf, 64, 10, 0.5, 0)
    rep = parity.stepwise_sampled_large(G, inst, eng, (0, 63), args.steps, seed=0)
    out["width_native"] = dict(rep, batch=64, n=inst.n, L=inst.L, seconds=time.perf_counter() - t0)
    eng.free()
    # the paper's form: k = 3 normalisation on the device, 32 members (W = 1)
    c3 = cnf.normalize(3)
    off, lits = c3.csr()
    inst3 = I.Instance("PL-k3", c3.n, off, lits)
    t0 = time.perf_counter()
    eng = G.Engine(c3, 32, 10, 0.5, 0)
    rep = parity.stepwise_sampled_large(G, inst3, eng, (0, 31), args.steps, seed=0)
    out["normalised_k3"] = dict(rep, batch=32, n=inst3.n, L=inst3.L, seconds=time.perf_counter() - t0)
    eng.free()
    c3.free()
    cnf.free()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
