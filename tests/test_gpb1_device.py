"""GPB1 bytes straight to a device table (pgpb_table_load_gpb1) vs the
reference's load_table + ArcTable path (table.py:250-310).

CPU: every malformed-file class the reference's load_table / validate
rejects is rejected by the native parser before any device work
(PGPB_EFORMAT).  GPU: tables loaded natively advance and decode bit for bit
like the ArcTable path, including a table written by the reference CLI's
build-tree (byte-identical to ours, tests/test_cli.py)."""

import ctypes
import struct

import numpy as np
import pytest

import gen_inputs as gi
from conftest import product_table


def _bytes(tab):
    import io

    from paper_2508_07014_b200 import save_table

    import tempfile
    from pathlib import Path

    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "t.gpb"
        save_table(tab, p)
        return p.read_bytes()


def _native(data: bytes):
    from paper_2508_07014_b200 import _lib

    h = ctypes.c_void_p()
    buf = ctypes.create_string_buffer(data, len(data)) if data else None
    rc = _lib.LIB.pgpb_table_load_gpb1(buf, len(data), 0, ctypes.byref(h))
    return rc, _lib.last_error()


@pytest.fixture(scope="module")
def fig_bytes():
    phrases = [[3, 1, 20], [3, 1, 20, 19], [3, 19, 22], [19, 9, 20]]
    return _bytes(product_table(phrases, 28))


def test_malformed_gpb1_rejected_without_device(fig_bytes):
    from paper_2508_07014_b200 import _lib

    good = bytearray(fig_bytes)
    S, V, A = struct.unpack_from("<III", good, 8)
    cases = {
        "truncated header": bytes(good[:10]),
        "bad magic": b"GPB2" + bytes(good[4:]),
        "unsupported version": bytes(good[:4]) + struct.pack("<I", 2) + bytes(good[8:]),
        "expected": bytes(good[:-1]),
    }
    arc_to = 24 + 2 * 4 * A
    bad_to = bytearray(good)
    struct.pack_into("<i", bad_to, arc_to, S + 5)
    cases["arc_to out of range"] = bytes(bad_to)
    tok = 24 + 4 * A
    bad_sort = bytearray(good)
    t0, t1 = struct.unpack_from("<ii", bad_sort, tok)
    struct.pack_into("<ii", bad_sort, tok, t1, t0)
    cases["sorted"] = bytes(bad_sort)
    bw = 24 + 16 * A + 12 * S  # backoff_weight f32[S]
    fin = 24 + 16 * A + 16 * S  # is_final u8[S]
    fin_states = [s for s in range(S) if good[fin + s]]
    nonfin = [s for s in range(1, S) if not good[fin + s]]
    pos_bw = bytearray(good)
    struct.pack_into("<f", pos_bw, bw + 4 * nonfin[0], 0.5)
    cases["non-final backoff weights must be <= 0"] = bytes(pos_bw)
    fin_bw = bytearray(good)
    struct.pack_into("<f", fin_bw, bw + 4 * fin_states[0], -1.0)
    cases["final states must have zero backoff weight"] = bytes(fin_bw)
    st_end = 24 + 16 * A + 4 * S
    st_start = 24 + 16 * A
    owner = max(range(S), key=lambda s: struct.unpack_from("<i", good, st_end + 4 * s)[0]
                - struct.unpack_from("<i", good, st_start + 4 * s)[0])
    short = bytearray(good)
    struct.pack_into("<i", short, st_end + 4 * owner, struct.unpack_from("<i", good, st_start + 4 * owner)[0])
    cases["arc ranges do not cover the arc array"] = bytes(short)
    nan_w = bytearray(good)
    struct.pack_into("<f", nan_w, 24 + 12 * A, float("nan"))
    cases["non-finite weight"] = bytes(nan_w)
    # a 45-byte file claiming V = 2^31 - 1 (must not abort the process)
    huge = bytearray(b"GPB1" + struct.pack("<IIIIf", 1, 1, 2**31 - 1, 0, 0.0) + bytes(21))
    cases["vocab_size"] = bytes(huge)
    for what, data in cases.items():
        rc, msg = _native(data)
        assert rc == _lib.PGPB_EFORMAT, what
        assert what.split()[0] in msg, (what, msg)


def test_native_validator_matches_load_table_messages(fig_bytes, tmp_path):
    """Same verdict and message as the reference-semantics load_table
    (table.py:267-310 -> validate :87-127) for every invariant class,
    including overlapping arc ranges (rejected without materialising S x A)."""
    from paper_2508_07014_b200 import TableFormatError, load_table

    good = bytearray(fig_bytes)
    S, V, A = struct.unpack_from("<III", good, 8)
    bw = 24 + 16 * A + 12 * S
    fin = 24 + 16 * A + 16 * S
    st_start, st_end = 24 + 16 * A, 24 + 16 * A + 4 * S
    variants = {}
    v = bytearray(good)
    struct.pack_into("<f", v, bw + 4 * [s for s in range(1, S) if not good[fin + s]][0], 0.25)
    variants["pos_backoff"] = v
    v = bytearray(good)
    for s in range(S):  # every state claims every arc
        struct.pack_into("<i", v, st_start + 4 * s, 0)
        struct.pack_into("<i", v, st_end + 4 * s, A)
    variants["overlap"] = v
    for name, data in variants.items():
        p = tmp_path / f"{name}.gpb"
        p.write_bytes(bytes(data))
        with pytest.raises(TableFormatError) as ei:
            load_table(p)
        rc, msg = _native(bytes(data))
        assert rc != 0
        assert msg in str(ei.value), (name, msg, str(ei.value))


def test_is_final_any_nonzero_byte_is_final(fig_bytes, tmp_path):
    """The reference reads is_final with astype(bool) (table.py:300): a byte
    of 7 on a final state is accepted, not rejected."""
    from paper_2508_07014_b200 import load_table

    good = bytearray(fig_bytes)
    S, V, A = struct.unpack_from("<III", good, 8)
    fin = 24 + 16 * A + 16 * S
    s = [i for i in range(S) if good[fin + i]][0]
    good[fin + s] = 7
    p = tmp_path / "f7.gpb"
    p.write_bytes(bytes(good))
    t = load_table(p)
    assert bool(t.is_final[s])
    rc, msg = _native(bytes(good))
    assert "is_final" not in msg


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["p20k_v1024", "p5k_v1024", "p20k_v4096"])
def test_device_loaded_table_advances_like_arctable(name, tmp_path):
    import torch

    from paper_2508_07014_b200 import get_scores_batch, load_table, load_table_device, save_table

    phrases, V = gi.corpus(name)
    tab = product_table(phrases, V)
    path = tmp_path / "t.gpb"
    save_table(tab, path)
    dt = load_table_device(path)
    assert (dt.num_states, dt.vocab_size, dt.num_arcs) == (tab.num_states, tab.vocab_size, tab.num_arcs)
    rng = np.random.default_rng(5)
    st = torch.from_numpy(rng.integers(0, tab.num_states, size=4096).astype(np.int32)).cuda()
    a = get_scores_batch(load_table(path), st)
    b = get_scores_batch(dt, st)
    assert torch.equal(a.scores.view(torch.int32), b.scores.view(torch.int32))
    assert torch.equal(a.next_states, b.next_states)
    dt2 = load_table_device(path.read_bytes())
    c = get_scores_batch(dt2, st.cpu().numpy())
    assert np.array_equal(c.next_states, b.next_states.cpu().numpy())


@pytest.mark.gpu
def test_device_loaded_table_decodes_like_arctable(tmp_path):
    from paper_2508_07014_b200 import DecodeConfig, ctc_greedy_boosted_batch, load_table_device, save_table

    phrases, V = gi.corpus("p20k_v1024")
    tab = product_table(phrases, V)
    path = tmp_path / "t.gpb"
    save_table(tab, path)
    dt = load_table_device(path)
    rng = np.random.default_rng(9)
    lps = np.stack([gi.random_emissions(rng, 120, V) for _ in range(16)])
    for lam in (0.5, 1.0):
        x = ctc_greedy_boosted_batch(lps, None, tab, DecodeConfig(lam=lam), blank_id=0, want_trace=True)
        y = ctc_greedy_boosted_batch(lps, None, dt, DecodeConfig(lam=lam), blank_id=0, want_trace=True)
        assert x == y


@pytest.mark.gpu
def test_malformed_file_raises_table_format_error(tmp_path):
    from paper_2508_07014_b200 import TableFormatError, load_table_device

    p = tmp_path / "bad.gpb"
    p.write_bytes(b"GPB1" + b"\0" * 30)
    with pytest.raises(TableFormatError):
        load_table_device(p)


@pytest.mark.gpu
@pytest.mark.parametrize("j", range(0, 16, 3))
def test_device_loaded_table_aed_beam_matches_reference_golden(j, tmp_path):
    """AED beam (eos bump on and off) with a table that exists only on the
    device: the bump's final part comes from the device arena
    (pgpb_final_bonus), same n-best as the reference golden."""
    from conftest import golden
    from test_beam_gpu import _cmp

    from paper_2508_07014_b200 import DecodeConfig, TableStepModel, aed_beam_boosted, load_table_device, save_table

    c = golden()["aed_beam"][j]
    rng = np.random.default_rng(c["seed"])
    phrases, V, c0, beta = gi.random_tree_spec(rng, max_phrases=10, max_len=4, max_vocab=12)
    tab = product_table(phrases, V, c0, beta)
    rows, default = gi.random_aed_rows(rng, V)
    model = TableStepModel(flavor="aed", default_row=default, rows=rows, eos_id=c["eos"])
    path = tmp_path / "t.gpb"
    save_table(tab, path)
    dt = load_table_device(path)
    best, nbest = aed_beam_boosted(model, dt, DecodeConfig(lam=c["lam"], beam_size=c["beam"],
                                                           eos_bump_enabled=c["eos_bump"]),
                                   max_len=c["max_len"], want_trace=True)
    _cmp(nbest, c["nbest"])
