"""Fused greedy kernels (GPU): bit-exact tokens, scores and traces.

CTC: pgpb_ctc_greedy vs golden reference outputs and the oracle; batched
calls equal per-utterance calls.  Transducer: pgpb_greedy_step through
transducer_greedy_boosted vs golden reference outputs and the oracle.
"""

import numpy as np
import pytest

import gen_inputs as gi
from conftest import golden, product_table, res_tuple
from test_oracle import aed_case, transducer_case  # noqa: F401

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _ctc_case(c):
    rng = np.random.default_rng(c["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=20, max_len=6, max_vocab=24)
    tab = product_table(phrases, V, c0, beta)
    T = int(rng.integers(3, 40))
    lp = gi.random_emissions(rng, T, V)
    assert gi.sha(lp) == c["lp_sha"]
    return tab, lp


@pytest.mark.parametrize("j", range(40))
def test_ctc_greedy_matches_reference_golden(j):
    from paper_2508_07014_b200 import DecodeConfig, EmissionMatrix, ctc_greedy_boosted

    c = golden()["ctc_greedy"][j]
    tab, lp = _ctc_case(c)
    r = ctc_greedy_boosted(EmissionMatrix(lp, blank_id=0), tab, DecodeConfig(lam=c["lam"]), want_trace=True)
    assert res_tuple(r) == c["result"]


def test_ctc_greedy_batch_equals_per_utterance_golden():
    from paper_2508_07014_b200 import DecodeConfig, ctc_greedy_boosted_batch

    # config 1: 100-phrase tree, V=1024, 4 x 200 frames
    phrases, V = gi.corpus("p100_v1024")
    tab = product_table(phrases, V)
    rng = np.random.default_rng(0)
    lps = np.stack([gi.random_emissions(rng, 200, V) for _ in range(4)])
    for lam in (0.0, 1.0):
        got = ctc_greedy_boosted_batch(lps, None, tab, DecodeConfig(lam=lam), blank_id=0, want_trace=True)
        exp = [c["result"] for c in golden()["config1"] if c["lam"] == lam]
        assert [res_tuple(r) for r in got] == exp


def test_ctc_greedy_ragged_batch_vs_oracle():
    from paper_2508_07014_b200 import DecodeConfig, ctc_greedy_boosted_batch

    phrases, V = gi.corpus("p20k_v1024")
    tab = product_table(phrases, V)
    rng = np.random.default_rng(11)
    B, T = 48, 120
    lps = np.stack([gi.random_emissions(rng, T, V) for _ in range(B)])
    lens = rng.integers(0, T + 1, size=B).astype(np.int32)
    lens[0] = T
    for lam in (0.0, 0.5, 1.0, 3.0):
        got = ctc_greedy_boosted_batch(lps, lens, tab, DecodeConfig(lam=lam), blank_id=0, want_trace=True)
        for b in range(B):
            e = orc.ctc_greedy_decode(lps[b, : lens[b]], 0, tab, lam)
            g = res_tuple(got[b])
            assert g["tokens"] == e["tokens"] and g["am"] == e["am"] and g["boost"] == e["boost"]
            assert g["trace"] == [list(x) for x in e["trace"]]


def test_ctc_greedy_20k_boosting_path_is_exercised():
    """Emissions built so the boosted rerank changes tokens; oracle-exact."""
    from paper_2508_07014_b200 import DecodeConfig, ctc_greedy_boosted_batch

    phrases, V = gi.corpus("p20k_v1024")
    tab = product_table(phrases, V)
    rng = np.random.default_rng(12)
    B, T = 16, 150
    logits = rng.normal(0, 0.3, size=(B, T, V))
    # make phrase tokens compete closely with the argmax
    for b in range(B):
        ph = phrases[int(rng.integers(len(phrases)))]
        for i, tok in enumerate(ph):
            logits[b, 2 * i + 1, tok] += 2.0
            logits[b, 2 * i + 1, (tok % (V - 1)) + 1] += 2.2
    lps = gi.log_softmax(logits).astype(np.float32)
    base = ctc_greedy_boosted_batch(lps, None, tab, DecodeConfig(lam=0.0), blank_id=0)
    got = ctc_greedy_boosted_batch(lps, None, tab, DecodeConfig(lam=1.0), blank_id=0, want_trace=True)
    changed = 0
    for b in range(B):
        e = orc.ctc_greedy_decode(lps[b], 0, tab, 1.0)
        g = res_tuple(got[b])
        assert g["tokens"] == e["tokens"] and g["am"] == e["am"] and g["boost"] == e["boost"]
        changed += base[b].tokens != got[b].tokens
    assert changed > 0


def test_lambda_zero_disabled_empty_identity():
    from paper_2508_07014_b200 import DecodeConfig, EmissionMatrix, ctc_greedy_boosted

    rng = np.random.default_rng(1004)
    for _ in range(20):
        V = int(rng.integers(4, 33))
        phrases = gi.random_phrase_set(rng, 6, 4, V)
        tab = product_table(phrases, V)
        empty = product_table([], V)
        em = EmissionMatrix(gi.random_emissions(rng, int(rng.integers(2, 51)), V), blank_id=0)
        a = ctc_greedy_boosted(em, tab, DecodeConfig(lam=0.0)).tokens
        b = ctc_greedy_boosted(em, tab, DecodeConfig(lam=1.0, boost_enabled=False)).tokens
        c = ctc_greedy_boosted(em, empty, DecodeConfig(lam=1.0)).tokens
        assert a == b == c


def test_ctc_errors(fig_table):
    from paper_2508_07014_b200 import DecodeConfig, EmissionMatrix, ctc_greedy_boosted

    rng = np.random.default_rng(2)
    em = EmissionMatrix(gi.random_emissions(rng, 4, 5), blank_id=0)
    with pytest.raises(ValueError, match="vocab size"):
        ctc_greedy_boosted(em, fig_table, DecodeConfig())
    em.blank_id = None
    with pytest.raises(ValueError, match="blank"):
        ctc_greedy_boosted(em, None, DecodeConfig())


@pytest.mark.parametrize("j", range(16))
def test_transducer_greedy_matches_reference_golden(j):
    from paper_2508_07014_b200 import DecodeConfig, TableStepModel, transducer_greedy_boosted

    c = golden()["transducer_greedy"][j]
    rng = np.random.default_rng(c["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=12)
    tab = product_table(phrases, V, c0, beta)
    rows, default = gi.random_transducer_rows(rng, V)
    model = TableStepModel(flavor="transducer", default_row=default, rows=rows)
    r = transducer_greedy_boosted(model, c["T"], 0, tab, DecodeConfig(lam=c["lam"], max_symbols_per_frame=c["cap"]),
                                  want_trace=True)
    assert res_tuple(r) == c["result"]


def test_greedy_step_kernel_vs_oracle_rerank():
    """pgpb_greedy_step on a [B,V] batch equals the reference rerank per row."""
    import torch

    from paper_2508_07014_b200 import _lib

    phrases, V = gi.corpus("p20k_v1024")
    tab = product_table(phrases, V)
    rng = np.random.default_rng(21)
    B = 512
    lp = gi.random_emissions(rng, B, V, scale=0.5)
    states = rng.integers(0, tab.num_states, size=B).astype(np.int32)
    d = lambda x: torch.from_numpy(x).cuda()  # noqa: E731
    ch = torch.empty(B, dtype=torch.int32, device="cuda")
    lpc = torch.empty(B, dtype=torch.float32, device="cuda")
    dl = torch.empty(B, dtype=torch.float64, device="cuda")
    nx = torch.empty(B, dtype=torch.int32, device="cuda")
    bl = torch.empty(B, dtype=torch.uint8, device="cuda")
    lpd, std = d(lp), d(states)
    for lam in (0.5, 1.0, 2.5):
        _lib.check(_lib.LIB.pgpb_greedy_step(tab.device_table().handle, lpd.data_ptr(), V, B, V, std.data_ptr(), None,
                                             0, lam, 1, ch.data_ptr(), lpc.data_ptr(), dl.data_ptr(), nx.data_ptr(),
                                             bl.data_ptr(), _lib.stream_ptr()))
        sc, nn = orc.score_batch(tab, states)
        chn, dln, nxn = ch.cpu().numpy(), dl.cpu().numpy(), nx.cpu().numpy()
        for b in range(B):
            a = int(np.argmax(lp[b]))
            if a == 0:
                assert bl[b].item() == 1
                continue
            e = orc._rerank(lp[b], sc[b], lam, (0,))
            assert chn[b] == e and dln[b] == float(sc[b, e]) and nxn[b] == nn[b, e]
