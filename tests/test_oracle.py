"""Pin the oracle (oracle/cgbn_oracle.py) before trusting it as the GPU checker.

(1) Frozen literals of the reference's own unit tests.
(2) Golden vectors produced by running the real reference (tests/golden/*.npz).
(3) The reference's algebraic invariants.
"""

import numpy as np
import pytest

from oracle import cgbn_oracle as O
from golden_cases import case_names, load_case


def test_frozen_bn_case():
    # test_batchnorm.py:86-97 — literals computed with scalar loops by the reference.
    rng = np.random.default_rng(23)
    x = rng.normal(size=(4, 2))
    st = O.RankState(gamma=[1.5, 0.5], beta=[0.1, -0.2])
    out = O.group_train_forward([x], [st])[0]
    assert abs(out["mu"][0] - 0.4591714964384243) < 1e-15
    assert abs(out["mu"][1] - -0.90541242423664) < 1e-15
    assert abs(out["var"][0] - 0.12006252582474286) < 1e-15
    assert abs(out["var"][1] - 1.7584970005300984) < 1e-15
    assert abs(out["y"][0, 0] - 0.5072946592418226) < 1e-12
    assert abs(out["y"][0, 1] - 0.22343109749756324) < 1e-12


def test_frozen_channel_sum_f64():
    # test_tensor.py:133-140
    rng = np.random.default_rng(17)
    x = rng.normal(size=(3, 2, 2, 2))
    cnt, s, _ = O.channel_sum(x)
    assert s[0] == 0.17595964399948189
    assert s[1] == -2.969076027521793
    assert cnt == 12


def test_frozen_channel_sum_f32():
    # test_tensor.py:148-156
    rng = np.random.default_rng(17)
    rng.normal(size=(3, 2, 2, 2))
    x32 = rng.normal(size=(4, 3)).astype(np.float32)
    _, s, _ = O.channel_sum(x32)
    assert s.dtype == np.float32
    assert float(s[0]) == 0.8578172326087952
    assert float(s[1]) == -2.2112133502960205
    assert float(s[2]) == -2.396543025970459


def test_sequential_sum_order_sensitivity():
    # test_tensor.py:98-104 — the left fold is the only acceptable answer.
    got = O.sequential_sum_rows(np.array([[1e16], [1.0], [-1e16]]))
    assert got[0] == 0.0


def test_star_allreduce_ascending_fold():
    # collectives.py:293-295; test_collectives.py:43-51 (−0.0 preserved: -0.0 + -0.0)
    v = [np.array([1e16, -0.0]), np.array([1.0, -0.0]), np.array([-1e16, -0.0])]
    out = O.star_allreduce(v)
    assert out[0] == 0.0
    assert np.signbit(out[1])


def test_bn_group_sums_collectives_fixture():
    # test_collectives.py:82-95: bn-group sums [3,3,12,12] for ranks holding rank+1
    vals = [np.array([float(r + 1)]) for r in range(4)]
    g0 = O.star_allreduce(vals[:2])
    g1 = O.star_allreduce(vals[2:])
    assert g0[0] == 3.0 and g1[0] == 7.0
    assert O.star_allreduce(vals)[0] == 10.0


@pytest.mark.parametrize("name", case_names())
def test_oracle_matches_reference_golden(name):
    meta, a = load_case(name)
    world, g = meta["world"], meta["bn_group"]
    xs = [a[f"x_{r}"].astype(np.float64) for r in range(world)]
    dys = [a[f"dy_{r}"].astype(np.float64) for r in range(world)]
    res = O.cgbn_world(xs, a["gamma"].astype(np.float64), a["beta"].astype(np.float64), g,
                       one_pass=meta["one_pass"], relu=meta["relu"], dys=dys,
                       eps=meta["eps"], momentum=meta["momentum"],
                       running=(a["running_mean0"].astype(np.float64),
                                a["running_var0"].astype(np.float64)))
    for r in range(world):
        for key in ("y", "mu", "var", "running_mean", "running_var", "dx", "dgamma", "dbeta",
                    "x_hat"):
            want = a[f"{key}_{r}"]
            got = res[r][key]
            assert O.rel_err(got, want) <= 1e-12, (name, r, key, O.rel_err(got, want))
        assert res[r]["m"] == int(a[f"m_{r}"])


@pytest.mark.parametrize("name", case_names())
def test_oracle_eval_matches_reference_golden(name):
    meta, a = load_case(name)
    from oracle.cgbn_oracle import RankState, eval_forward
    rm = a["running_mean_0"].astype(np.float32).astype(np.float64)
    rv = a["running_var_0"].astype(np.float32).astype(np.float64)
    st = RankState(a["gamma"].astype(np.float64), a["beta"].astype(np.float64), meta["eps"],
                   rm, rv, meta["momentum"])
    got = eval_forward(a["x_0"].astype(np.float64), st)
    assert O.rel_err(got, a["eval_y_0"]) <= 1e-13


def test_concat_equivalence_invariant():
    # test_batchnorm.py:190-217: CGBN == local BN on the rank-ordered concatenation
    rng = np.random.default_rng(40)
    for world, g in [(2, 2), (4, 4), (4, 2), (3, 3), (6, 3)]:
        c = int(rng.integers(1, 5))
        shards = [rng.normal(size=(int(rng.integers(1, 5)), c, 2, 3)) for _ in range(world)]
        gamma = rng.uniform(0.5, 1.5, c)
        beta = rng.normal(size=c)
        res = O.cgbn_world(shards, gamma, beta, g)
        for gi in range(world // g):
            members = range(gi * g, (gi + 1) * g)
            ref = O.cgbn_world([np.concatenate([shards[r] for r in members])], gamma, beta, 1)[0]
            got = np.concatenate([res[r]["y"] for r in members])
            assert np.allclose(got, ref["y"], rtol=1e-9, atol=1e-12)


def test_small_count_rejected():
    # batchnorm.py:133-137 / test_batchnorm.py:110-113
    with pytest.raises(ValueError, match="at least 2"):
        O.group_train_forward([np.ones((1, 3))], [O.RankState(np.ones(3), np.zeros(3))])


@pytest.mark.parametrize("relu,shapes", [
    (False, [(3, 10, 4, 5), (2, 10, 4, 5)]),
    (True, [(4, 7, 3, 3)] * 3),
    (False, [(6, 9)] * 2),
])
def test_group_blocks_matches_literal_restatement(relu, shapes):
    """The memory-bounded block oracle (used at bench sizes) agrees with the literal
    restatement group_train_forward / group_backward to ~1e-12."""
    rng = np.random.default_rng(5)
    c = shapes[0][1]
    xs = [rng.normal(loc=2.0, size=s) for s in shapes]
    dys = [rng.normal(size=s) for s in shapes]
    gamma, beta = rng.uniform(0.5, 1.5, c), rng.normal(size=c)
    g = len(shapes)
    ref = O.cgbn_world(xs, gamma, beta, g, relu=relu, dys=dys)
    outs = list(O.group_blocks(xs, gamma, beta, dys=dys, relu=relu, block_elems=40))
    assert len(outs) > 1  # several channel blocks
    for b in outs:
        c0, c1 = b["c0"], b["c1"]
        for key in ("mu", "var", "running_mean", "running_var", "dgamma", "dbeta"):
            assert O.rel_err(b[key], ref[0][key][c0:c1]) <= 1e-12, key
        assert b["m"] == ref[0]["m"]
        for r in range(g):
            assert O.rel_err(b["y"][r], ref[r]["y"][:, c0:c1]) <= 1e-12
            assert O.rel_err(b["dx"][r], ref[r]["dx"][:, c0:c1]) <= 1e-12
