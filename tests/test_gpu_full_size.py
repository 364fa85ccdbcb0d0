"""Oracle parity of the production kernels at BASELINE.json's full sizes (-m gpu).

The engines run in the launch configuration bench.py times (non-debug kernels, the fused
forward + check sweep driven by enqueue, lanes where the bench uses them, the sweep's chunk
loop where the X/R slices exceed its L2 budget). The oracle cannot step a million-variable
batch, but members are independent and draw their random numbers from counters of their
GLOBAL index (R1, R2), so sampled members are recomputed one by one: before every
step the sampled members' fp32 iterates are read in place (galois_engine_get_member) and
handed to the oracle (exact map, reading R24), and each step is compared with the one-step
bounds (tests/parity.py stepwise_sampled). A debug engine adds the signal G (bit-exact) and
g1 (relative 1e-5) of the sampled members.
"""
import numpy as np
import pytest

from paper_2603_28796_b200 import instances as I
from tests import parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2603_28796_b200 import galois
    galois.lib()
    return galois


@pytest.fixture(scope="module")
def c4():
    return I.CONFIGS["C4"][0]()


@pytest.fixture(scope="module")
def c5():
    return I.CONFIGS["C5"][0]()


C4_MEMBERS = (0, 1, 31, 32, 517, 1000, 1023)


def test_c4_production_stepwise(G, c4):
    """configs[3] (1M variables, 4.2M clauses, widths 2-30, power-law occurrences, hubs up
    to ~200k occurrences, a 2 GB E buffer), B = 1024 as the bench runs it: 3 steps of the
    fused sweep, hub partials and k_update_tma<0,...> on sampled members."""
    deg = I.degrees(c4)
    assert deg.max() > 100_000                      # hub chunks take part
    cnf = G.Cnf.from_instance(c4)
    eng = G.Engine(cnf, 1024, 50, 0.5, 0)
    rep = parity.stepwise_sampled(G, c4, eng, C4_MEMBERS, 3, seed=0)
    assert rep["compared"] >= len(C4_MEMBERS) * 3 - 2, rep
    eng.free()
    cnf.free()


def test_c4_debug_signal(G, c4):
    """The same instance on a debug engine: G of every variable of the sampled members is
    the oracle's exactly (hub partials included), g1 within 1e-5 relative."""
    cnf = G.Cnf.from_instance(c4)
    eng = G.Engine(cnf, 1024, 5, 0.5, 0, debug=True)
    ties = parity.debug_signal_sampled(G, c4, eng, C4_MEMBERS, seed=0)
    assert ties <= 1
    eng.free()
    cnf.free()


C5_MEMBERS = (0, 1023, 1024, 4100, 6143, 8191)


def test_c5_chunk_loop_stepwise(G, c5):
    """configs[4]'s instance (100k variables, 16 cube pins) at 8192 members per GPU: the X/R
    slices of the eight 1024-member chunks (25.6 MB each) exceed the sweep's 48 MB L2 budget,
    so the staged sweep k_sweep_tma<..., kLoop = true> walks the chunks in a loop (the
    instantiation C5 runs at every GPU count); sampled members from several chunks, pins
    forced."""
    cnf = G.Cnf.from_instance(c5)
    eng = G.Engine(cnf, 8192, 50, 0.5, 0, cubes=c5.pins)
    rep = parity.stepwise_sampled(G, c5, eng, C5_MEMBERS, 3, seed=0, cubes=c5.pins)
    assert rep["compared"] >= len(C5_MEMBERS) * 3 - 2, rep
    eng.free()
    cnf.free()


def test_c5_chunk_loop_debug_signal(G, c5):
    cnf = G.Cnf.from_instance(c5)
    eng = G.Engine(cnf, 8192, 5, 0.5, 0, cubes=c5.pins, debug=True)
    ties = parity.debug_signal_sampled(G, c5, eng, C5_MEMBERS, seed=0, cubes=c5.pins)
    assert ties <= 1
    eng.free()
    cnf.free()


def test_chunk_loop_wide_tiles_stepwise(G):
    """k_sweep_tma's other index path: 200k variables (X/R slices of 51 MB: the chunk loop)
    and clause widths up to 40, so the width-sorted tail has 32-clause tiles of more than
    512 slots, which read their slots from global memory instead of the staged tile;
    B = 2048 (two chunks), sampled members of both, 3 steps."""
    inst = I.industrial(200_000, 120_000, 7, wmin=2, wmax=40, width_exp=1.2)
    w = np.diff(inst.offsets)
    assert (w >= 17).sum() >= 64                    # whole tiles past the 512-slot stage
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, 2048, 20, 0.5, 0)
    members = (0, 5, 1023, 1024, 1500, 2047)
    rep = parity.stepwise_sampled(G, inst, eng, members, 3, seed=0)
    assert rep["compared"] >= len(members) * 3 - 2, rep
    eng.free()
    cnf.free()


@pytest.mark.parametrize("batch,pinned", [(1024, False), (2048, False), (1024, True)])
def test_pair_update_odd_n_stepwise(G, batch, pinned):
    """The production update over variable pairs (k_update_pair): an odd variable count
    (the last pair has one variable), hubs, degrees past one 56-row piece (such pairs go
    variable by variable) and pairs that travel as one stage; B = 1024 stages the two rows
    of a pair with one copy per array, B = 2048 with two. With `pinned`, cube pins on the
    two highest-degree (hub) variables and on two low-degree ones whose pair partner is
    free. Sampled members, 4 steps."""
    inst = I.industrial(2501, 30_000, 21, occ_exp=0.9)
    deg = I.degrees(inst)
    assert inst.n % 2 == 1 and (deg > 256).any() and ((deg > 56) & (deg <= 256)).any()
    pins = ()
    if pinned:
        low = [v for v in range(0, inst.n - 1, 2) if 0 < deg[v] <= 8][:2]     # 0-based, even: pair heads
        pins = tuple(sorted(set(I.top_degree_vars(inst, 2)) | {v + 1 for v in low}))
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, batch, 20, 0.5, 0, cubes=pins)
    members = (0, 3, 511, 700, batch - 1)
    rep = parity.stepwise_sampled(G, inst, eng, members, 4, seed=0, cubes=pins)
    assert rep["compared"] >= len(members) * 4 - 2, rep
    eng.free()
    cnf.free()


@pytest.mark.parametrize("batch,pinned", [(32, False), (64, True), (128, False), (256, True), (512, False)])
def test_small_window_update_stepwise(G, batch, pinned):
    """The production update of sub-1024 batches (k_update_smallw: groups of 32 / W
    variables per item, E rows of W words staged by bulk copy, hub rows skipped for the
    hub partials; f4's windows on instances too large for 1024 resident members): an
    odd variable count (a ragged last group), hubs, degrees past one 16 KB piece at W = 16,
    cube pins on hub and low-degree variables. Sampled members incl. the last, 4 steps."""
    inst = I.industrial(2501, 30_000, 21, occ_exp=0.9)
    deg = I.degrees(inst)
    assert inst.n % 2 == 1 and (deg > 256).any()
    pins = ()
    if pinned:
        low = [v for v in range(inst.n) if 0 < deg[v] <= 8][:2]
        pins = tuple(sorted(set(I.top_degree_vars(inst, 2)) | {v + 1 for v in low}))
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, batch, 20, 0.5, 0, cubes=pins)
    members = tuple(sorted({0, 3, batch // 2 + 1, batch - 1}))
    rep = parity.stepwise_sampled(G, inst, eng, members, 4, seed=0, cubes=pins)
    assert rep["compared"] >= len(members) * 4 - 2, rep
    eng.free()
    cnf.free()


def test_stepwise_large_harness(G):
    """The per-variable tie harness that tools/pl_parity.py runs at the paper's largest size
    (stepwise_sampled_large), on a small instance in the same kernel configuration (64
    members: k_update_smallw + the fused scalar sweep)."""
    inst = I.industrial_large(30_000, 120_000, 3)
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, 64, 10, 0.5, 0)
    rep = parity.stepwise_sampled_large(G, inst, eng, (0, 63), 3)
    assert rep["member_steps"] == 6 and rep["compared_vars"] > 0.9 * 6 * inst.n, rep
    eng.free()
    cnf.free()


def test_c2_lanes_stepwise(G):
    """configs[1] (B = 4096) split into the bench's 4 lanes (4 streams): sampled members of
    every lane, 4 steps."""
    inst = I.CONFIGS["C2"][0]()
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, 4096, 50, 0.5, 0, lanes=4)
    members = (0, 1023, 1024, 2047, 2500, 3072, 4095)
    rep = parity.stepwise_sampled(G, inst, eng, members, 4, seed=0)
    assert rep["compared"] >= len(members) * 4 - 2, rep
    eng.free()
    cnf.free()


@pytest.mark.parametrize("which", ["C3a", "C3b"])
def test_c3_wide_stepwise(G, which):
    """configs[2]: 5-SAT n = 2000 (average degree 105: the bit-sliced signal counts) and
    7-SAT n = 500 (the sweep's wide shape, hub partials for every variable), B = 16384 in
    the bench's 2 lanes; sampled members, 2 steps."""
    inst = I.CONFIGS[which][0]()
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, 16384, 50, 0.5, 0, lanes=2)
    members = (0, 4097, 8191, 8192, 16383)
    rep = parity.stepwise_sampled(G, inst, eng, members, 2, seed=0)
    assert rep["compared"] >= len(members) * 2 - 2, rep
    eng.free()
    cnf.free()
