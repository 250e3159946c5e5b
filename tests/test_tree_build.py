"""Host-side tree compilation (libpgpb C++) is array-identical to the reference (CPU).

Pinned against golden vectors produced by the reference itself, and against
the reference's known-answer values (tests/test_tree.py:25-34, :179-194,
tests/test_table.py:23-40 of the reference suite).
"""

import math

import numpy as np
import pytest

import gen_inputs as gi
from conftest import golden, golden_npz, golden_tree_case, product_table

from paper_2508_07014_b200 import (ArcTable, ContextList, Phrase, TableFormatError, TreeParams, Vocabulary,
                                   arc_score, build_prefix_tree, compile_arc_table, compute_fail_links,
                                   context_list_from_texts, load_table, naive_score, save_table, state_strings,
                                   tokenize)
from paper_2508_07014_b200.errors import TokenizationError, VocabularyError

FIELDS = ["arc_from", "arc_token", "arc_to", "arc_weight", "state_start", "state_end", "backoff_to",
          "backoff_weight", "is_final", "final_score", "root_scores", "root_next"]

FIG_DUMP = (
    "0\t''\tdepth=0\tarc=0.000000\tacc=0.000000\tfinal=F\tfail=0\n"
    "1\t'c'\tdepth=1\tarc=1.000000\tacc=1.000000\tfinal=F\tfail=0\n"
    "7\t's'\tdepth=1\tarc=1.000000\tacc=1.000000\tfinal=F\tfail=0\n"
    "2\t'ca'\tdepth=2\tarc=2.693147\tacc=3.693147\tfinal=F\tfail=0\n"
    "5\t'cs'\tdepth=2\tarc=2.693147\tacc=3.693147\tfinal=F\tfail=7\n"
    "8\t'si'\tdepth=2\tarc=2.693147\tacc=3.693147\tfinal=F\tfail=0\n"
    "3\t'cat'\tdepth=3\tarc=3.098612\tacc=6.791759\tfinal=T\tfail=0\n"
    "6\t'csv'\tdepth=3\tarc=3.098612\tacc=6.791759\tfinal=T\tfail=0\n"
    "9\t'sit'\tdepth=3\tarc=3.098612\tacc=6.791759\tfinal=T\tfail=0\n"
    "4\t'cats'\tdepth=4\tarc=3.386294\tacc=10.178054\tfinal=T\tfail=7\n"
)


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype.kind == "f":
        return a.shape == b.shape and np.array_equal(a.view(np.uint8), np.asarray(b, a.dtype).view(np.uint8))
    return np.array_equal(a, b.astype(a.dtype) if a.dtype != b.dtype else b)


@pytest.mark.parametrize("i", range(40))
def test_tables_bit_identical_to_reference(i):
    g, phrases, V, c0, beta, unk, _ = golden_tree_case(i)
    z = golden_npz()
    tree, tab = product_table(phrases, V, c0, beta, g["mode"], g["bonus"], unk, with_tree=True)
    for f in FIELDS:
        assert bits_equal(getattr(tab, f), z[f"tree{i}_{f}"]), f
    assert bits_equal(tree.acc_scores, z[f"tree{i}_acc"])
    if g["dump"] is not None:
        assert tree.dump() == g["dump"]


@pytest.mark.parametrize("name", list(gi.CORPORA))
def test_corpus_tables_bit_identical_to_reference(name):
    g = golden()["corpora"][name]
    phrases, V = gi.corpus(name)
    tree, tab = product_table(phrases, V, with_tree=True)
    assert (tab.num_states, tab.num_arcs, tree.max_depth) == (g["S"], g["A"], g["max_depth"])
    for f in FIELDS:
        assert gi.sha(np.asarray(getattr(tab, f))) == g["arrays"][f], f


def test_fig1_golden_dump_and_values(fig_tree, fig_table, letters_vocab):
    assert fig_tree.dump(letters_vocab) == FIG_DUMP
    names = {fig_tree.node_string(n, letters_vocab): n for n in range(fig_tree.num_nodes)}
    for d, exp in ((1, 1.0), (2, 2.6931), (3, 3.0986), (4, 3.3863)):
        assert arc_score(d, TreeParams()) == pytest.approx(exp, abs=1e-4)
    assert fig_tree.acc_scores[names["cat"]] == pytest.approx(6.7917, abs=1e-4)
    assert float(fig_table.backoff_weight[names["ca"]]) == pytest.approx(-3.6931, abs=1e-4)
    assert float(fig_table.backoff_weight[names["cs"]]) == pytest.approx(-2.6931, abs=1e-4)
    assert int(fig_table.backoff_to[names["cs"]]) == names["s"]
    for w in ("cat", "cats", "csv", "sit"):
        assert fig_table.backoff_weight[names[w]] == 0.0 and fig_table.is_final[names[w]]
    assert fig_table.num_arcs == 9
    # R1 golden numbering
    assert [names[s] for s in ("c", "ca", "cat", "cats", "cs", "csv", "s", "si", "sit")] == list(range(1, 10))


def test_nodes_view_matches_reference_structure(fig_tree, letters_vocab):
    nodes = fig_tree.nodes
    c = letters_vocab.id_of("c")
    assert nodes[0].arcs[c][0] == 1 and nodes[1].parent == 0 and nodes[1].in_token == c
    assert nodes[4].fail == 7 and nodes[3].is_final
    assert fig_tree.bfs_order() == [0, 1, 7, 2, 5, 8, 3, 6, 9, 4]


def test_naive_score_known_answers(fig_tree, letters_vocab):
    n = {fig_tree.node_string(i, letters_vocab): i for i in range(fig_tree.num_nodes)}
    ids = {ch: letters_vocab.id_of(ch) for ch in "ctix"}
    assert naive_score(fig_tree, 0, ids["c"]) == (1.0, n["c"])
    s, x = naive_score(fig_tree, n["ca"], ids["t"])
    assert s == pytest.approx(3.0986, abs=1e-4) and x == n["cat"]
    s, x = naive_score(fig_tree, n["cs"], ids["i"])
    assert s == pytest.approx(0.0, abs=1e-6) and x == n["si"]
    with pytest.raises(IndexError):
        naive_score(fig_tree, fig_tree.num_nodes, 0)


def test_build_errors_match_reference(letters_vocab):
    ctx = ContextList(phrases=[Phrase("ok", (1, 2)), Phrase("bad", (1, 99))], min_chars=0)
    with pytest.raises(ValueError, match="token id 99 out of range for V=28"):
        build_prefix_tree(ctx, TreeParams(), 28)
    with pytest.raises(ValueError, match="empty phrase"):
        build_prefix_tree(ContextList(phrases=[Phrase("e", ())], min_chars=0), TreeParams(), 28)
    tree = build_prefix_tree(context_list_from_texts(["cat"], letters_vocab), TreeParams(), letters_vocab.size)
    with pytest.raises(ValueError, match="fail links"):
        compile_arc_table(tree)
    with pytest.raises(ValueError):
        TreeParams(c0=-1)
    with pytest.raises(ValueError):
        TreeParams(weight_mode="bogus")


def test_uniform_bonus_positive_backoff_is_rejected_like_reference():
    # a non-final state failing to a single-token final with a bonus gets a
    # positive backoff; the reference's compile-time validate() raises
    with pytest.raises(TableFormatError, match="non-final backoff"):
        product_table([(2,), (1, 2, 3)], 8, mode="uniform", bonus=1.5)


def test_empty_context_list():
    tab = product_table([], 7, unk=0.25)
    assert tab.num_states == 1 and tab.num_arcs == 0
    assert (tab.root_scores == np.float32(0.25)).all() and (tab.root_next == 0).all()


def test_gpb1_round_trip_and_errors(fig_table, tmp_path):
    p = tmp_path / "f.gpb"
    save_table(fig_table, p)
    t2 = load_table(p)
    for f in FIELDS:
        assert bits_equal(getattr(t2, f), getattr(fig_table, f)), f
    q = tmp_path / "g.gpb"
    save_table(t2, q)
    assert p.read_bytes() == q.read_bytes()
    blob = p.read_bytes()
    p.write_bytes(blob[:-7])
    with pytest.raises(TableFormatError, match="bytes"):
        load_table(p)
    bad = bytearray(blob)
    bad[:4] = b"NOPE"
    p.write_bytes(bytes(bad))
    with pytest.raises(TableFormatError, match="magic"):
        load_table(p)
    bad = bytearray(blob)
    bad[4] = 99
    p.write_bytes(bytes(bad))
    with pytest.raises(TableFormatError, match="version"):
        load_table(p)
    bad = bytearray(blob)
    bad[24:28] = (9999).to_bytes(4, "little")
    p.write_bytes(bytes(bad))
    with pytest.raises(TableFormatError, match="corrupt"):
        load_table(p)


def test_gpb1_byte_identical_to_reference_layout(tmp_path):
    # header "<4sIIIIf" + A*16 + S*21 bytes (table.py:16-29, :279)
    tab = product_table([(1, 2, 3), (2, 3)], 5)
    p = tmp_path / "t.gpb"
    save_table(tab, p)
    assert len(p.read_bytes()) == 24 + 16 * tab.num_arcs + 21 * tab.num_states


def test_state_strings(fig_tree, fig_table, letters_vocab):
    labels = state_strings(fig_table, letters_vocab)
    for i in range(fig_tree.num_nodes):
        assert labels[i] == fig_tree.node_string(i, letters_vocab)


def test_context_and_vocab(letters_vocab):
    assert tokenize("cab", letters_vocab) == [3, 1, 2]
    with pytest.raises(TokenizationError):
        tokenize("c4t", letters_vocab)
    ctx = context_list_from_texts(["ab", "cat", "cat", "dog"], letters_vocab)
    assert ctx.texts == ["cat", "dog"]
    v = Vocabulary(tokens=tuple(f"t{i}" for i in range(8)))
    assert tokenize("7 3", v, mode="ids") == [7, 3]
    with pytest.raises(TokenizationError):
        tokenize("9", v, mode="ids")
    with pytest.raises(VocabularyError):
        Vocabulary(tokens=("a", "a"))
    with pytest.raises(VocabularyError):
        Vocabulary(tokens=("a", "b"), blank_id=0, eos_id=0)


def test_validate_catches_corruption(fig_table):
    import copy

    t = copy.copy(fig_table)
    t.backoff_weight = fig_table.backoff_weight.copy()
    t.backoff_weight[1] = 0.5
    with pytest.raises(TableFormatError, match="non-final"):
        t.validate()
    t = copy.copy(fig_table)
    t.arc_token = fig_table.arc_token[::-1].copy()
    with pytest.raises(TableFormatError):
        t.validate()
