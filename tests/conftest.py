"""Shared fixtures.  `-m gpu` tests need a CUDA device; everything else runs on CPU."""

from __future__ import annotations

import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
for p in (str(ROOT), str(HERE)):
    if p not in sys.path:
        sys.path.insert(0, p)

import gen_inputs as gi  # noqa: E402

LETTERS = "abcdefghijklmnopqrstuvwxyz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_cuda = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_cuda = False
    if has_cuda:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@lru_cache(maxsize=1)
def golden() -> dict:
    return json.loads((HERE / "golden" / "golden.json").read_text())


@lru_cache(maxsize=1)
def golden_npz():
    return dict(np.load(HERE / "golden" / "golden.npz"))


@pytest.fixture
def letters_vocab():
    from paper_2508_07014_b200.context import Vocabulary

    return Vocabulary(tokens=("<b>",) + tuple(LETTERS) + (" ",), blank_id=0)


@pytest.fixture
def fig_tree(letters_vocab):
    from paper_2508_07014_b200 import TreeParams, build_prefix_tree, compute_fail_links, context_list_from_texts

    ctx = context_list_from_texts(["cat", "cats", "csv", "sit"], letters_vocab)
    return compute_fail_links(build_prefix_tree(ctx, TreeParams(), letters_vocab.size))


@pytest.fixture
def fig_table(fig_tree):
    from paper_2508_07014_b200 import compile_arc_table

    return compile_arc_table(fig_tree, unk_score=0.0)


def product_table(phrases, V, c0=1.0, beta=2.0, mode="depth_scaled", bonus=0.0, unk=0.0, with_tree=False):
    """Product tree build from token-id phrases (ContextList order)."""
    from paper_2508_07014_b200 import (ContextList, Phrase, TreeParams, build_prefix_tree, compile_arc_table,
                                       compute_fail_links)

    ctx = ContextList(phrases=[Phrase(" ".join(map(str, p)), tuple(p)) for p in phrases], min_chars=0)
    tree = compute_fail_links(build_prefix_tree(ctx, TreeParams(c0, beta, mode, bonus), V))
    tab = compile_arc_table(tree, unk_score=unk)
    return (tree, tab) if with_tree else tab


def golden_tree_case(i):
    g = golden()["trees"][i]
    rng = np.random.default_rng(g["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=50, max_len=8, max_vocab=64)
    unk = float(rng.choice([0.0, 0.3, -0.2]))
    assert gi.phrases_sha(phrases) == g["phrases_sha"], "input generator drifted"
    return g, phrases, V, c0, beta, unk, rng


def res_tuple(r):
    """DecodeResult -> comparable dict in the golden format."""
    return {"tokens": [int(x) for x in r.tokens], "am": float(r.am_score), "boost": float(r.boost_score),
            "trace": [[int(s.token), float(s.boost), int(s.state)] for s in (r.trace or [])]}
