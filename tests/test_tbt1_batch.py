"""TBT1 files straight to a device batch (acoustic.load_emissions_batch) vs
the per-file reference loader (acoustic.py:84-130): same values, same
validation errors (header/shape errors of any file are reported before
normalisation errors, which the batch checks on the GPU)."""

import numpy as np
import pytest

import gen_inputs as gi

pytestmark = pytest.mark.gpu


def _files(tmp_path, rng, n=7, V=33):
    from paper_2508_07014_b200 import EmissionMatrix, save_emissions

    paths = []
    for i in range(n):
        lp = gi.random_emissions(rng, int(rng.integers(1, 60)), V)
        p = tmp_path / f"e{i}.tbt"
        save_emissions(EmissionMatrix(lp, blank_id=0), p)
        paths.append(p)
    return paths


def test_batch_equals_per_file_loader(tmp_path):
    from paper_2508_07014_b200 import load_emissions
    from paper_2508_07014_b200.acoustic import load_emissions_batch

    paths = _files(tmp_path, np.random.default_rng(1))
    lp, lens = load_emissions_batch(paths)
    lp, lens = lp.cpu().numpy(), lens.cpu().numpy()
    for i, p in enumerate(paths):
        em = load_emissions(p)
        assert lens[i] == em.num_frames
        assert np.array_equal(lp[i, : lens[i]].view(np.uint32), em.logprobs.view(np.uint32))
        assert not lp[i, lens[i]:].any()


def test_batch_validation_errors(tmp_path):
    from paper_2508_07014_b200 import EmissionFormatError, EmissionMatrix, save_emissions
    from paper_2508_07014_b200.acoustic import load_emissions_batch

    paths = _files(tmp_path, np.random.default_rng(2), n=3)
    bad = tmp_path / "bad.tbt"
    save_emissions(EmissionMatrix(np.zeros((4, 33), np.float32)), bad)  # rows not normalised
    with pytest.raises(EmissionFormatError, match="bad.tbt: rows not log-normalized"):
        load_emissions_batch(paths + [bad])
    with pytest.warns(UserWarning):
        load_emissions_batch(paths + [bad], strict=False)
    trunc = tmp_path / "trunc.tbt"
    trunc.write_bytes(paths[0].read_bytes()[:-4])
    with pytest.raises(EmissionFormatError, match="payload bytes"):
        load_emissions_batch([trunc])
    other = tmp_path / "v.tbt"
    save_emissions(EmissionMatrix(gi.random_emissions(np.random.default_rng(0), 5, 12)), other)
    with pytest.raises(EmissionFormatError, match="vocab size"):
        load_emissions_batch(paths + [other])
