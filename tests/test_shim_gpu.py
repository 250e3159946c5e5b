"""kernels_shim: the reference `_kernels` contract served by the B200 kernels (GPU).

Compared with the reference's own compiled Cython module (oracle/_ref,
built from /root/reference and shipped with the snapshot) when present,
otherwise with the oracle's C restatement.
"""

import numpy as np
import pytest

import gen_inputs as gi

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _ref():
    return orc.ref_kernels() or type("O", (), {
        "score_batch": staticmethod(lambda *a: orc.lib() and _oracle_score(*a)),
        "ctc_greedy": staticmethod(lambda lp, b, lam, u, *arr: _oracle_ctc(lp, b, lam, u, *arr)),
    })


class _T:
    def __init__(self, arrs, V):
        (self.arc_token, self.arc_to, self.arc_weight, self.state_start, self.state_end, self.backoff_to,
         self.backoff_weight, self.root_scores, self.root_next) = arrs
        self.vocab_size = V


def _oracle_score(*a):
    *arrs, st = a
    return orc.score_batch(_T(arrs, arrs[7].shape[0]), st)


def _oracle_ctc(lp, blank, lam, use, *arrs):
    return orc.ctc_greedy(lp, blank, lam, use, _T(arrs, arrs[7].shape[0]))


def test_shim_score_batch_and_ctc_greedy_equal_reference_kernels():
    from paper_2508_07014_b200 import kernels_shim as ks

    ref = _ref()
    rng = np.random.default_rng(100)
    for _ in range(15):
        phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=40, max_len=8, max_vocab=64)
        t = orc.build_table(phrases, V, c0, beta, unk=float(rng.uniform(-0.5, 0.5)))
        arrs = orc._tab_arrays(t)
        st = rng.integers(0, t.num_states, size=int(rng.integers(1, 40))).astype(np.int32)
        a = ks.score_batch(*arrs, st)
        b = ref.score_batch(*arrs, st)
        assert np.array_equal(a[0].view(np.uint32), b[0].view(np.uint32)) and np.array_equal(a[1], b[1])
        lp = gi.random_emissions(rng, int(rng.integers(3, 40)), V)
        for lam in (0.0, 0.3, 1.0, 2.0):
            x = ks.ctc_greedy(lp, 0, lam, lam != 0, *arrs)
            y = ref.ctc_greedy(lp, 0, lam, lam != 0, *arrs)
            assert np.array_equal(x[0], y[0]) and x[1] == y[1] and x[2] == y[2]
            assert np.array_equal(x[3], y[3]) and np.array_equal(x[4], y[4])


def test_shim_error_conventions():
    from paper_2508_07014_b200 import kernels_shim as ks

    t = orc.build_table([(1, 2)], 4)
    arrs = orc._tab_arrays(t)
    with pytest.raises(ValueError, match="dtype"):
        ks.score_batch(*arrs, np.array([0], np.int64))
    with pytest.raises(ValueError, match="C-contiguous"):
        ks.score_batch(*arrs, np.array([0, 0, 0, 0], np.int32)[::2])
    s, n = ks.score_batch(*arrs, np.zeros(0, np.int32))
    assert s.shape == (0, 4) and n.shape == (0, 4)
