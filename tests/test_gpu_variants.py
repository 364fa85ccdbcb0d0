"""The execution variants against the oracle DIRECTLY (-m gpu): the single-launch run of
small instances (k_small_run), CUDA-graph replay of 8-step chunks, lanes (with graphs), and
sub-batch windows (f4) — each driven through galois_engine_run, the call a user makes, and
compared with the fp64 oracle run over the same steps (tests/parity.py oracle_multistep):
rc and stop step, the best record (u*, t*, b*) and its bits, every member's last count, and
the final iterate within north_star's trajectory bound 1e-4 max(1, |z|).

Where the variants start from an injected iterate (set_iterate at t0) the two sides share
it exactly; free-running fp32 against fp64 can only part at a decision that comes within
the accumulated rounding of its threshold, so members whose oracle trajectory has such a
near tie (|a| or |z| within 2e-5 max(1, |z|)) are counted and excepted from the
member-wise checks.
"""
import numpy as np
import pytest

from oracle import oracle as O
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


def _iterate(B, n, t, seed=1):
    rng = np.random.default_rng(seed)
    z = (rng.normal(size=(B, n)) * 2.5).astype(np.float32)
    m = (rng.normal(size=(B, n)) * 0.3).astype(np.float32)
    v = (np.abs(rng.normal(size=(B, n))) * 0.2).astype(np.float32)
    return z, m, v


def _init_state(G, cnf, inst, B, T, seed, **kw):
    """The engine's own initial iterate (a3) for the oracle: z0 from an engine of the same
    seed (RNG counters of the global member index make it the same for any variant)."""
    e = G.Engine(cnf, B, T, 0.5, seed, **kw)
    z, m, v, t = e.get_iterate()
    e.free()
    assert t == 0
    return O.State.from_reduced(z, m, v, 0)


@pytest.mark.parametrize("seed", [0, 2, 5])
def test_small_run_first_sat_vs_oracle(G, seed):
    """configs[0] (3-SAT n = 50, m = 213, B = 1024, 100 steps) through run(): one launch of
    k_small_run (cooperative grid barrier at every check) against the oracle's run from the
    same initial iterate, t = 0 check included."""
    inst = I.random_ksat(50, 213, 3, seed)
    cnf = G.Cnf.from_instance(inst)
    st = _init_state(G, cnf, inst, 1024, 100, 0)
    eng = G.Engine(cnf, 1024, 100, 0.5, 0)
    res = parity.compare_run_variant(G, inst, eng, parity.oracle_cfg(0), st, 100, check_t0=True, max_near=40)
    eng.free()
    cnf.free()
    print(res)


@pytest.mark.parametrize("K", [1, 3])
def test_small_run_from_injected_iterate(G, K):
    """k_small_run from an identical injected iterate at t0 = 20 to T = 45 (checks every K)."""
    inst = I.random_ksat(50, 213, 3, 7)
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, 1024, 45, 0.5, 3, check_interval=K)
    z, m, v = _iterate(1024, inst.n, 20)
    eng.set_iterate(z, m, v, 20)
    st = O.State.from_reduced(z, m, v, 20)
    res = parity.compare_run_variant(G, inst, eng, parity.oracle_cfg(3), st, 45, K=K, max_near=60)
    eng.free()
    cnf.free()
    print(res)


@pytest.mark.parametrize("K,B", [(1, 2048), (3, 3000)])
def test_graph_replay_vs_oracle(G, K, B):
    """CUDA graphs forced (galois_engine_set_graphs(1)): 8-step (K = 1) or 6-step (K = 3)
    chunks captured once and replayed from t0 = 8 (kernel parameters frozen at capture, step
    index read on the device) to T = 41 (a direct-launch tail)."""
    inst = I.random_ksat(200, 852, 3, 3)
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, B, 41, 0.5, 4, check_interval=K, graphs=1)
    z, m, v = _iterate(B, inst.n, 8, seed=2)
    eng.set_iterate(z, m, v, 8)
    st = O.State.from_reduced(z, m, v, 8)
    res = parity.compare_run_variant(G, inst, eng, parity.oracle_cfg(4), st, 41, K=K, max_near=B // 4)
    eng.free()
    cnf.free()
    print(res)


@pytest.mark.parametrize("lanes,graphs", [(4, 1), (2, 0)])
def test_lanes_vs_oracle(G, lanes, graphs):
    """The bench's lanes (4 concurrent engines on their own streams, CUDA-graph chunks) from
    one injected iterate at t0 = 8 to T = 40."""
    inst = I.random_ksat(200, 852, 3, 4)
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, 4096, 40, 0.5, 6, lanes=lanes, graphs=graphs)
    z, m, v = _iterate(4096, inst.n, 8, seed=3)
    eng.set_iterate(z, m, v, 8)
    st = O.State.from_reduced(z, m, v, 8)
    res = parity.compare_run_variant(G, inst, eng, parity.oracle_cfg(6), st, 40, max_near=1024)
    eng.free()
    cnf.free()
    print(res)


def test_lanes_first_sat_vs_oracle(G):
    """Lanes with a SAT stop: the record and its bits equal the oracle's (other lanes may run
    past t*, so only the record, the stop and the counts are compared)."""
    inst = I.random_ksat(50, 213, 3, 0)
    cnf = G.Cnf.from_instance(inst)
    st = _init_state(G, cnf, inst, 4096, 100, 0)
    eng = G.Engine(cnf, 4096, 100, 0.5, 0, lanes=4)
    res = parity.compare_run_variant(G, inst, eng, parity.oracle_cfg(0), st, 100, check_t0=True,
                                     compare_state=False, max_near=160, counts_after_sat=False)
    assert res["rc"] == G.SAT
    eng.free()
    cnf.free()


@pytest.mark.parametrize("K,sub", [(1, 1024), (3, 992), (1, 256), (2, 64)])
def test_windows_vs_oracle(G, K, sub):
    """f4 sub-batching: 3000 members in windows of `sub`, each run from t = 0; the
    best record over the windows, the bits and every member's last count against the
    oracle's run of the whole batch from the same initial iterate."""
    inst = I.random_ksat(120, 510, 3, 8)
    cnf = G.Cnf.from_instance(inst)
    st = _init_state(G, cnf, inst, 3000, 24, 1)
    eng = G.Engine(cnf, 3000, 24, 0.5, 1, check_interval=K, sub_batch=sub)
    res = parity.compare_run_variant(G, inst, eng, parity.oracle_cfg(1), st, 24, K=K, check_t0=True,
                                     compare_state=False, max_near=600, counts_after_sat=False)
    eng.free()
    cnf.free()
    print(res)


@pytest.mark.parametrize("world,B", [(2, 1000), (3, 100)])
def test_rank_slices_equal_one_gpu_and_oracle(G, world, B):
    """Row e's sharding without the transport: `world` engines each running one rank's slice
    (set_comm with no communicator — same slices, global member indices and RNG counters as
    the NCCL path) merged by the exchange's key, lexicographic min (u, t, b), equal the
    single engine's record and bits, and that engine's run equals the oracle's. B = 100 at
    world 3 leaves the last rank with no members (b_per = 64)."""
    inst = I.random_ksat(120, 510, 3, 8)
    cnf = G.Cnf.from_instance(inst)
    T = 24
    st = _init_state(G, cnf, inst, B, T, 1)
    one = G.Engine(cnf, B, T, 0.5, 1)
    z_one = one.get_iterate()[0]
    parity.compare_run_variant(G, inst, one, parity.oracle_cfg(1), st, T, check_t0=True, compare_state=False,
                               max_near=200, counts_after_sat=False)
    best1 = one.best_assignment()
    counts1, _ = one.unsat_counts()
    b_per = -(-(-(-B // world)) // 32) * 32
    recs = []
    for r in range(world):
        e = G.Engine(cnf, B, T, 0.5, 1, rank=r, world=world)
        lo, hi = min(B, r * b_per), min(B, (r + 1) * b_per)
        z = e.get_iterate()[0]
        np.testing.assert_array_equal(z[:hi - lo], z_one[lo:hi])       # global RNG counters
        e.run()
        if hi > lo:
            b = e.best_assignment()
            assert lo <= b["global_b"] < hi
            recs.append(((b["unsat"], b["step"], b["global_b"]), b["values"]))
            if best1["unsat"] > 0:                                       # no SAT stop anywhere
                c, first = e.unsat_counts()
                assert first == lo
                np.testing.assert_array_equal(c[:hi - lo], counts1[lo:hi])
        e.free()
    key, values = min(recs, key=lambda kv: kv[0])
    assert key == (best1["unsat"], best1["step"], best1["global_b"])
    np.testing.assert_array_equal(values, best1["values"])
    one.free()
    cnf.free()


def test_nccl_single_rank_vs_oracle(G):
    """The NCCL exchange path (1-rank communicator: MIN all-reduce and the global record on
    the exchange stream, winner broadcast) against the oracle from one injected iterate."""
    inst = I.random_ksat(200, 852, 3, 5)
    cnf = G.Cnf.from_instance(inst)
    eng = G.Engine(cnf, 2048, 40, 0.5, 2, rank=0, world=1, nccl_id=G.galois_comm_unique_id())
    z, m, v = _iterate(2048, inst.n, 8, seed=4)
    eng.set_iterate(z, m, v, 8)
    st = O.State.from_reduced(z, m, v, 8)
    res = parity.compare_run_variant(G, inst, eng, parity.oracle_cfg(2), st, 40, max_near=512)
    eng.free()
    cnf.free()
    print(res)
