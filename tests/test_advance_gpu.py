"""Advance kernel parity (GPU): bit-exact scores and next states.

Checked against (a) golden vectors from the reference implementation,
(b) the CPU oracle (C restatement of _kernels.pyx:30-72) on fresh seeded
inputs up to the benchmark sizes, and (c) size-independent properties.
"""

import threading

import numpy as np
import pytest

import gen_inputs as gi
from conftest import golden, golden_npz, golden_tree_case, product_table

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("i", range(40))
def test_advance_matches_reference_golden(i):
    from paper_2508_07014_b200 import get_scores_batch

    g, phrases, V, c0, beta, unk, _ = golden_tree_case(i)
    z = golden_npz()
    tab = product_table(phrases, V, c0, beta, g["mode"], g["bonus"], unk)
    res = get_scores_batch(tab, z[f"tree{i}_states"])
    assert res.scores.dtype == np.float32 and res.next_states.dtype == np.int32
    assert bits_equal(res.scores, z[f"tree{i}_scores"])
    assert np.array_equal(res.next_states, z[f"tree{i}_next"])


@pytest.mark.parametrize("name", list(gi.CORPORA))
def test_advance_corpora_match_reference_golden(name):
    import torch

    from paper_2508_07014_b200 import get_scores_batch

    g = golden()["corpora"][name]
    phrases, V = gi.corpus(name)
    tab = product_table(phrases, V)
    states = np.random.default_rng(99).integers(0, tab.num_states, size=512).astype(np.int32)
    assert gi.sha(states) == g["advance_states_sha"]
    res = get_scores_batch(tab, states)
    assert gi.sha(res.scores) == g["advance_scores_sha"]
    assert gi.sha(res.next_states) == g["advance_next_sha"]
    for b, v, s, n in g["cells"]:
        assert float(res.scores[b, v]) == s and int(res.next_states[b, v]) == n
    # device-tensor path and the chain-walk variant agree bit for bit
    d = get_scores_batch(tab, torch.from_numpy(states).cuda())
    assert bits_equal(d.scores.cpu().numpy(), res.scores)
    assert np.array_equal(d.next_states.cpu().numpy(), res.next_states)
    from paper_2508_07014_b200.table import _advance_device

    c = _advance_device(tab, torch.from_numpy(states).cuda(), check=True, out=None, chain=True)
    assert bits_equal(c.scores.cpu().numpy(), res.scores)
    assert np.array_equal(c.next_states.cpu().numpy(), res.next_states)


@pytest.mark.parametrize("chain,single", [(False, 0), (False, 2), (True, 0)])
@pytest.mark.parametrize("name,B", [("p20k_v1024", 8192), ("p20k_v4096", 2048), ("p5k_v1024", 3000),
                                    ("p20k_v1024", 37), ("p20k_v1024", 1024), ("p20k_v1024", 65)])
def test_advance_full_size_vs_oracle(name, B, chain, single):
    """The production advance (small batches through the blob kernel at one
    step, the single-advance kernel otherwise or when forced by the tuning
    key), and the reference chain-walk kernel, bit-exact against the oracle
    at the benchmark sizes."""
    import torch

    from paper_2508_07014_b200 import _lib
    from paper_2508_07014_b200.table import _advance_device

    phrases, V = gi.corpus(name)
    tab = product_table(phrases, V)
    rng = np.random.default_rng(B)
    states = rng.integers(0, tab.num_states, size=B).astype(np.int32)
    _lib.set_tuning("adv.compact", single)
    try:
        d = _advance_device(tab, torch.from_numpy(states).cuda(), check=True, out=None, chain=chain)
    finally:
        _lib.set_tuning("adv.compact", 0)
    sc, nx = orc.score_batch(tab, states)
    assert bits_equal(d.scores.cpu().numpy(), sc)
    assert np.array_equal(d.next_states.cpu().numpy(), nx)


def _closure_biased_tokens(tab, states0, R, rng, p_closure=0.6):
    """Token stream for R chained steps where about p_closure of the steps
    take a first-hit (closure) arc of the current state, so the successor
    lookup exercises the entry path, not only the dense root row."""
    V = tab.vocab_size
    toks = np.empty((R, states0.size), np.int32)
    s = states0.copy()
    for k in range(R):
        sc, nx = orc.score_batch(tab, s)
        for b in range(s.size):
            over = np.nonzero(nx[b] != tab.root_next)[0] if rng.random() < p_closure else np.empty(0)
            toks[k, b] = int(rng.choice(over)) if over.size else int(rng.integers(0, V))
        s = nx[np.arange(s.size), toks[k]].astype(np.int32)
    return toks


@pytest.mark.parametrize("name,B,R,parts", [("p20k_v1024", 1024, 6, 0), ("p20k_v1024", 1024, 4, 1),
                                            ("p20k_v1024", 300, 5, 2), ("p20k_v1024", 97, 3, 8),
                                            ("p20k_v1024", 8192, 2, 0), ("p20k_v4096", 256, 3, 0),
                                            ("p5k_v1024", 4, 7, 0)])
@pytest.mark.parametrize("layout", [0, 1, 2, 3])
def test_advance_steps_vs_oracle(name, B, R, parts, layout):
    """Chained R-step advance (config 5): every step's rows bit-exact vs the
    oracle advance of that step's states, and s_{k+1} = next_k[b, tok_k[b]]."""
    import torch

    from paper_2508_07014_b200 import advance_steps

    phrases, V = gi.corpus(name)
    tab = product_table(phrases, V)
    rng = np.random.default_rng(B * 31 + R)
    s0 = rng.integers(0, tab.num_states, size=B).astype(np.int32)
    if B <= 1024:
        toks = _closure_biased_tokens(tab, s0, R, rng)
    else:
        toks = rng.integers(0, V, size=(R, B)).astype(np.int32)
    from paper_2508_07014_b200 import _lib
    _lib.set_tuning("adv.compact", layout)  # 0 by regime, 1 ranked bitmap, 2 compact arrays, 3 blobs
    try:
        r = advance_steps(tab, torch.from_numpy(s0).cuda(), torch.from_numpy(toks).cuda(), parts=parts)
    finally:
        _lib.set_tuning("adv.compact", 0)
    tr = r.trace.cpu().numpy()
    assert np.array_equal(tr[0], s0)
    s = s0
    for k in range(R):
        assert np.array_equal(tr[k], s), f"step {k} states"
        sc, nx = orc.score_batch(tab, s)
        assert bits_equal(r.scores[k].cpu().numpy(), sc), f"step {k} scores"
        assert np.array_equal(r.next_states[k].cpu().numpy(), nx), f"step {k} next"
        s = nx[np.arange(B), toks[k]].astype(np.int32)
    assert np.array_equal(r.final_states.cpu().numpy(), s)


@pytest.mark.parametrize("V", [130, 28])
def test_advance_steps_generic_path(V):
    """Vocabularies the chained kernel cannot split (V % 128 != 0) take R
    single-step launches plus a successor gather: same contract."""
    import torch

    from paper_2508_07014_b200 import advance_steps

    rng = np.random.default_rng(V)
    tab = product_table(gi.random_phrase_set(rng, 40, 8, V), V, unk=0.1)
    B, R = 33, 4
    s0 = rng.integers(0, tab.num_states, size=B).astype(np.int32)
    toks = _closure_biased_tokens(tab, s0, R, rng)
    r = advance_steps(tab, torch.from_numpy(s0).cuda(), torch.from_numpy(toks).cuda())
    s = s0
    for k in range(R):
        sc, nx = orc.score_batch(tab, s)
        assert np.array_equal(r.trace[k].cpu().numpy(), s)
        assert bits_equal(r.scores[k].cpu().numpy(), sc) and np.array_equal(r.next_states[k].cpu().numpy(), nx)
        s = nx[np.arange(B), toks[k]].astype(np.int32)
    assert np.array_equal(r.final_states.cpu().numpy(), s)


def test_advance_steps_edge_cases(fig_table):
    import torch

    from paper_2508_07014_b200 import advance_steps

    z = torch.zeros(0, dtype=torch.int32, device="cuda")
    r = advance_steps(fig_table, z, torch.zeros((3, 0), dtype=torch.int32, device="cuda"))
    assert r.scores.shape == (3, 0, fig_table.vocab_size)
    with pytest.raises(IndexError):
        advance_steps(fig_table, torch.tensor([0], device="cuda"),
                      torch.tensor([[fig_table.vocab_size]], device="cuda"))
    with pytest.raises(ValueError):
        advance_steps(fig_table, torch.tensor([0, 1], device="cuda"), torch.tensor([[1]], device="cuda"))


def test_advance_properties_at_64k_rows():
    """Size-independent checks at B=65536 (512 MiB of output): every row of the
    same state is identical, and rows agree with a small oracle sample."""
    import torch

    from paper_2508_07014_b200 import get_scores_batch

    phrases, V = gi.corpus("p20k_v1024")
    tab = product_table(phrases, V)
    rng = np.random.default_rng(5)
    uniq = rng.integers(0, tab.num_states, size=64).astype(np.int32)
    states = torch.from_numpy(np.tile(uniq, 1024)).cuda()
    d = get_scores_batch(tab, states)
    s = d.scores.view(1024, 64, V)
    n = d.next_states.view(1024, 64, V)
    assert bool((s == s[:1]).all()) and bool((n == n[:1]).all())
    sc, nx = orc.score_batch(tab, uniq)
    assert bits_equal(s[0].cpu().numpy(), sc) and np.array_equal(n[0].cpu().numpy(), nx)


@pytest.mark.parametrize("V", [5, 7, 31, 33, 130])
def test_advance_odd_vocab_scalar_path(V):
    from paper_2508_07014_b200 import get_scores_batch

    rng = np.random.default_rng(V)
    for _ in range(5):
        phrases = gi.random_phrase_set(rng, 40, 8, V)
        unk = float(rng.uniform(-0.5, 0.5))
        tab = product_table(phrases, V, float(rng.uniform(0.1, 2)), float(rng.uniform(0, 3)), unk=unk)
        st = rng.integers(0, tab.num_states, size=int(rng.integers(1, 50))).astype(np.int32)
        r = get_scores_batch(tab, st)
        sc, nx = orc.score_batch(tab, st)
        assert bits_equal(r.scores, sc) and np.array_equal(r.next_states, nx)


def test_fig1_known_cells(fig_tree, fig_table, letters_vocab):
    from paper_2508_07014_b200 import get_scores_batch

    n = {fig_tree.node_string(i, letters_vocab): i for i in range(fig_tree.num_nodes)}
    ids = {ch: letters_vocab.id_of(ch) for ch in "catsvix"}
    r = get_scores_batch(fig_table, [0, n["ca"], n["cs"], n["cat"]])
    assert r.scores[0, ids["c"]] == pytest.approx(1.0) and r.next_states[0, ids["c"]] == n["c"]
    assert r.scores[1, ids["t"]] == pytest.approx(3.0986, abs=1e-4) and r.next_states[1, ids["t"]] == n["cat"]
    assert r.scores[1, ids["x"]] == pytest.approx(-3.6931, abs=1e-4) and r.next_states[1, ids["x"]] == 0
    assert r.scores[2, ids["i"]] == pytest.approx(0.0, abs=1e-6) and r.next_states[2, ids["i"]] == n["si"]
    assert r.scores[3, ids["x"]] == pytest.approx(0.0) and r.next_states[3, ids["x"]] == 0


def test_edge_cases(fig_table):
    import torch

    from paper_2508_07014_b200 import get_scores_batch

    r = get_scores_batch(fig_table, [])
    assert r.scores.shape == (0, fig_table.vocab_size)
    with pytest.raises(IndexError):
        get_scores_batch(fig_table, [fig_table.num_states])
    with pytest.raises(IndexError):
        get_scores_batch(fig_table, [-1])
    with pytest.raises(IndexError):
        get_scores_batch(fig_table, torch.tensor([99], device="cuda"))
    empty = product_table([], 28, unk=0.25)
    r = get_scores_batch(empty, [0, 0])
    assert (r.scores == np.float32(0.25)).all() and (r.next_states == 0).all()


def test_telescoping_and_neutralisation(fig_table, letters_vocab):
    from paper_2508_07014_b200 import get_scores_batch

    total, state = 0.0, 0
    for ch in "ca":
        r = get_scores_batch(fig_table, [state])
        total += float(r.scores[0, letters_vocab.id_of(ch)])
        state = int(r.next_states[0, letters_vocab.id_of(ch)])
    r = get_scores_batch(fig_table, [state])
    x = letters_vocab.id_of("x")
    total += float(r.scores[0, x])
    assert int(r.next_states[0, x]) == 0 and total == pytest.approx(fig_table.unk_score, abs=1e-5)


def test_concurrent_queries_are_isolated(fig_table):
    from concurrent.futures import ThreadPoolExecutor

    from paper_2508_07014_b200 import get_scores_batch

    rng = np.random.default_rng(77)
    batches = [rng.integers(0, fig_table.num_states, size=16) for _ in range(32)]
    expected = [get_scores_batch(fig_table, b) for b in batches]
    with ThreadPoolExecutor(max_workers=8) as pool:
        got = list(pool.map(lambda b: get_scores_batch(fig_table, b), batches * 4))
    for i, r in enumerate(got):
        e = expected[i % 32]
        assert bits_equal(r.scores, e.scores) and np.array_equal(r.next_states, e.next_states)


def test_row_max_matches_oracle():
    from paper_2508_07014_b200.table import ArcTable  # noqa: F401

    phrases, V = gi.corpus("p5k_v1024")
    tab = product_table(phrases, V)
    rm = tab.device_table().row_max().cpu().numpy()
    idx = np.random.default_rng(3).integers(0, tab.num_states, size=300)
    sc, _ = orc.score_batch(tab, idx.astype(np.int32))
    assert bits_equal(rm[idx], sc.max(axis=1))


@pytest.mark.parametrize("V,parts", [(896, 0), (512, 0), (512, 2), (256, 1), (128, 1)])
@pytest.mark.parametrize("layout", [0, 1, 2, 3])
def test_advance_steps_split_shapes(V, parts, layout):
    """Chained kernels at vocabularies below 1024 (compact arrays built, fewer
    than 32 bitmap words, one or two column parts; V = 896 leaves lanes 28-31
    without a word), every table layout, closure-biased token streams."""
    import torch

    from paper_2508_07014_b200 import _lib, advance_steps

    rng = np.random.default_rng(V * 7 + parts)
    tab = product_table(gi.random_phrase_set(rng, 300, 8, V), V, unk=-0.1)
    B, R = 77, 5
    s0 = rng.integers(0, tab.num_states, size=B).astype(np.int32)
    toks = _closure_biased_tokens(tab, s0, R, rng)
    _lib.set_tuning("adv.compact", layout)
    try:
        r = advance_steps(tab, torch.from_numpy(s0).cuda(), torch.from_numpy(toks).cuda(), parts=parts)
    finally:
        _lib.set_tuning("adv.compact", 0)
    s = s0
    for k in range(R):
        sc, nx = orc.score_batch(tab, s)
        assert np.array_equal(r.trace[k].cpu().numpy(), s)
        assert bits_equal(r.scores[k].cpu().numpy(), sc) and np.array_equal(r.next_states[k].cpu().numpy(), nx)
        s = nx[np.arange(B), toks[k]].astype(np.int32)
    assert np.array_equal(r.final_states.cpu().numpy(), s)


def test_advance_without_blobs_falls_back():
    """A state whose closure has >= 64 first-hit arcs (a root child with 100
    children) leaves the advance blobs unbuilt: single and chained advances
    then run on the compact arrays and stay bit-exact."""
    import torch

    from paper_2508_07014_b200 import advance_steps

    V = 256
    phrases = [(1, v) for v in range(2, 102)] + [(3, 4, 5), (7, 8)]
    tab = product_table(phrases, V)
    assert tab.device_table().info().max_closure >= 64
    rng = np.random.default_rng(64)
    B, R = 300, 4
    s0 = rng.integers(0, tab.num_states, size=B).astype(np.int32)
    toks = _closure_biased_tokens(tab, s0, R, rng)
    r = advance_steps(tab, torch.from_numpy(s0).cuda(), torch.from_numpy(toks).cuda())
    s = s0
    for k in range(R):
        sc, nx = orc.score_batch(tab, s)
        assert bits_equal(r.scores[k].cpu().numpy(), sc) and np.array_equal(r.next_states[k].cpu().numpy(), nx)
        s = nx[np.arange(B), toks[k]].astype(np.int32)
    from paper_2508_07014_b200.table import _advance_device

    d = _advance_device(tab, torch.from_numpy(s0).cuda(), check=True, out=None)
    sc, nx = orc.score_batch(tab, s0)
    assert bits_equal(d.scores.cpu().numpy(), sc) and np.array_equal(d.next_states.cpu().numpy(), nx)
