"""Weighted token trie with Aho-Corasick failure links (tree compilation, stage 1).

API mirror of the reference's `phraseboost.tree`
(/root/reference/pkg/src/phraseboost/tree.py).  The difference is the
representation: the reference keeps a list of `TreeNode` objects with
per-node dicts; here the trie is a set of flat arrays (parent, depth,
in_token, is_final, arc score, accumulated score, fail) produced by the
native builder in libpgpb (csrc/pgpb_tree.cpp), which is what the arc-table
compiler and the device layout consume.  `PrefixTree.nodes` materialises
reference-style `TreeNode` objects on demand for callers that walk them.

Node numbering is the reference's (creation order while inserting phrases
in ContextList order, tree.py:153-172), so state ids — and therefore the
advance kernel's next_states — are bit-identical.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .context import ContextList, Vocabulary

WEIGHT_DEPTH_SCALED = "depth_scaled"
WEIGHT_UNIFORM = "uniform"
WEIGHT_MODES = (WEIGHT_DEPTH_SCALED, WEIGHT_UNIFORM)
_MODE_CODE = {WEIGHT_DEPTH_SCALED: 0, WEIGHT_UNIFORM: 1}


@dataclass(frozen=True)
class TreeParams:
    """c0, beta and weight mode (tree.py:35-50)."""

    c0: float = 1.0
    beta: float = 2.0
    weight_mode: str = WEIGHT_DEPTH_SCALED
    uniform_final_bonus: float = 0.0

    def __post_init__(self):
        if self.c0 < 0:
            raise ValueError(f"c0 must be >= 0, got {self.c0}")
        if self.beta < 0:
            raise ValueError(f"beta must be >= 0, got {self.beta}")
        if self.weight_mode not in WEIGHT_MODES:
            raise ValueError(f"weight_mode must be one of {WEIGHT_MODES}, got {self.weight_mode!r}")


def arc_score(depth: int, params: TreeParams) -> float:
    """Score of the arc entering a node at `depth` (tree.py:53-61)."""
    if depth < 1:
        raise ValueError(f"arc depth must be >= 1, got {depth}")
    if params.weight_mode == WEIGHT_UNIFORM or depth == 1:
        return params.c0
    return params.c0 * params.beta + math.log(depth)


@dataclass
class TreeNode:
    """Reference-style node view (tree.py:64-74)."""

    id: int
    depth: int
    parent: int
    in_token: int | None
    arcs: dict[int, tuple[int, float]] = field(default_factory=dict)
    acc_score: float = 0.0
    is_final: bool = False
    fail: int | None = None


class PrefixTree:
    """Array-backed phrase trie; node 0 is the root."""

    def __init__(self, params: TreeParams, vocab_size: int, parent, depth, in_token, is_final,
                 arc_scores, acc_scores, fail=None):
        self.params = params
        self.vocab_size = int(vocab_size)
        self.parent = parent
        self.depth = depth
        self.in_token = in_token
        self.is_final = is_final
        self.arc_scores = arc_scores
        self.acc_scores = acc_scores
        self.fail = fail
        self._nodes: list[TreeNode] | None = None
        self._children: tuple[np.ndarray, np.ndarray] | None = None

    # -- reference PrefixTree surface (tree.py:77-142) ----------------------
    @property
    def num_nodes(self) -> int:
        return int(self.parent.shape[0])

    @property
    def num_finals(self) -> int:
        return int(self.is_final.sum())

    @property
    def max_depth(self) -> int:
        return int(self.depth.max())

    @property
    def has_fail_links(self) -> bool:
        return self.fail is not None

    def children(self) -> tuple[np.ndarray, np.ndarray]:
        """CSR (start[n+1], child ids) with children in ascending token order."""
        if self._children is None:
            n = self.num_nodes
            kids = np.arange(1, n, dtype=np.int64)
            order = np.lexsort((self.in_token[1:], self.parent[1:]))
            kids = kids[order]
            counts = np.bincount(self.parent[1:], minlength=n) if n > 1 else np.zeros(n, np.int64)
            start = np.zeros(n + 1, dtype=np.int64)
            np.cumsum(counts, out=start[1:])
            self._children = (start, kids)
        return self._children

    @property
    def nodes(self) -> list[TreeNode]:
        if self._nodes is None:
            start, kids = self.children()
            out = []
            for i in range(self.num_nodes):
                arcs = {
                    int(self.in_token[c]): (int(c), float(self.arc_scores[c]))
                    for c in kids[start[i]:start[i + 1]]
                }
                out.append(TreeNode(
                    id=i,
                    depth=int(self.depth[i]),
                    parent=int(self.parent[i]),
                    in_token=None if i == 0 else int(self.in_token[i]),
                    arcs=arcs,
                    acc_score=float(self.acc_scores[i]),
                    is_final=bool(self.is_final[i]),
                    fail=None if self.fail is None else int(self.fail[i]),
                ))
            self._nodes = out
        return self._nodes

    def arc_score_of(self, node_id: int) -> float:
        return 0.0 if node_id == 0 else float(self.arc_scores[node_id])

    def token_path(self, node_id: int) -> list[int]:
        ids: list[int] = []
        cur = int(node_id)
        while cur > 0:
            ids.append(int(self.in_token[cur]))
            cur = int(self.parent[cur])
        ids.reverse()
        return ids

    def node_string(self, node_id: int, vocab: Vocabulary | None = None) -> str:
        ids = self.token_path(node_id)
        if vocab is not None:
            return "".join(vocab.tokens[i] for i in ids)
        return ",".join(str(i) for i in ids)

    def bfs_order(self) -> list[int]:
        start, kids = self.children()
        order = [0]
        head = 0
        while head < len(order):
            nid = order[head]
            head += 1
            order.extend(int(c) for c in kids[start[nid]:start[nid + 1]])
        return order

    def dump(self, vocab: Vocabulary | None = None) -> str:
        """Listing of every node in BFS order, format of tree.py:132-142."""
        rows = []
        for nid in self.bfs_order():
            fail = None if self.fail is None else int(self.fail[nid])
            rows.append(
                f"{nid}\t'{self.node_string(nid, vocab)}'\tdepth={int(self.depth[nid])}"
                f"\tarc={self.arc_score_of(nid):.6f}\tacc={float(self.acc_scores[nid]):.6f}"
                f"\tfinal={'T' if self.is_final[nid] else 'F'}\tfail={fail}"
            )
        return "\n".join(rows) + "\n"

    def lookup(self, node_id: int, token: int) -> int:
        """Child of `node_id` on `token`, or -1."""
        start, kids = self.children()
        seg = kids[start[node_id]:start[node_id + 1]]
        toks = self.in_token[seg]
        i = int(np.searchsorted(toks, token))
        return int(seg[i]) if i < seg.shape[0] and toks[i] == token else -1


def build_prefix_tree(ctx: ContextList, params: TreeParams, vocab_size: int) -> PrefixTree:
    """Trie of the context list with depth-scaled/uniform scores (tree.py:145-186)."""
    phrases = ctx.phrases
    lens = np.fromiter((len(p.token_ids) for p in phrases), dtype=np.int64, count=len(phrases))
    offsets = np.zeros(len(phrases) + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    total = int(offsets[-1])
    tokens = np.fromiter((t for p in phrases for t in p.token_ids), dtype=np.int64, count=total)
    if total and (tokens.min() < -(2**31) or tokens.max() >= 2**31):
        tokens = np.clip(tokens, -1, vocab_size)  # out of int32: report as out of range below
    tokens = tokens.astype(np.int32)
    cap = total + 1
    parent = np.empty(cap, np.int32)
    depth = np.empty(cap, np.int32)
    in_token = np.empty(cap, np.int32)
    is_final = np.empty(cap, np.uint8)
    arc_sc = np.empty(cap, np.float64)
    acc = np.empty(cap, np.float64)
    n = _lib.c_int64(0)
    bad_p = _lib.c_int64(-1)
    bad_t = _lib.c_int64(-1)
    rc = _lib.LIB.pgpb_trie_build(
        _lib.ptr(tokens), _lib.ptr(offsets), len(phrases), int(vocab_size), float(params.c0),
        float(params.beta), _MODE_CODE[params.weight_mode], float(params.uniform_final_bonus), cap,
        _lib.ptr(parent), _lib.ptr(depth), _lib.ptr(in_token), _lib.ptr(is_final), _lib.ptr(arc_sc),
        _lib.ptr(acc), _lib.ctypes.byref(n), _lib.ctypes.byref(bad_p), _lib.ctypes.byref(bad_t),
    )
    if rc == _lib.PGPB_EINVAL and bad_p.value >= 0:
        ph = phrases[bad_p.value]
        if not ph.token_ids:
            raise ValueError(f"empty phrase {ph.text!r}")
        bad = next(t for t in ph.token_ids if not 0 <= t < vocab_size)
        raise ValueError(f"phrase {ph.text!r}: token id {bad} out of range for V={vocab_size}")
    _lib.check(rc, "pgpb_trie_build")
    k = n.value
    return PrefixTree(
        params, vocab_size, parent[:k].copy(), depth[:k].copy(), in_token[:k].copy(),
        is_final[:k].astype(bool), arc_sc[:k].copy(), acc[:k].copy(),
    )


def compute_fail_links(tree: PrefixTree) -> PrefixTree:
    """Aho-Corasick fail links, BFS with ascending tokens (tree.py:189-214); in place."""
    fail = np.empty(tree.num_nodes, np.int32)
    _lib.check(
        _lib.LIB.pgpb_trie_fail_links(
            tree.num_nodes, _lib.ptr(tree.parent), _lib.ptr(tree.in_token), tree.vocab_size,
            _lib.ptr(fail),
        ),
        "pgpb_trie_fail_links",
    )
    tree.fail = fail
    tree._nodes = None
    return tree
