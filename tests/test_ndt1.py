"""SURVEY 8(f)3 host side: NDT1 files (nds_read_tensor / nds_write_tensor vs the reference's
tensor_file.cpp, both directions, plus its rejection rules) and the reference generator
(nds_random_ode_system vs rng.cpp, bitwise). CPU only: these entry points need no device."""
import struct

import numpy as np
import pytest

import paper_2412_15840_b200 as nds


def _rand(rng, dims):
    return rng.standard_normal(dims) + 1j * rng.standard_normal(dims)


@pytest.mark.parametrize("dims", [(3,), (4, 5), (2, 3, 4), (1, 7, 1, 2), (2,) * 9])
def test_roundtrip_and_reference_compatibility(tmp_path, ref, dims):
    x = _rand(np.random.default_rng(len(dims)), dims)
    p_ours, p_ref = str(tmp_path / "ours.ndt"), str(tmp_path / "ref.ndt")
    nds.write_tensor(p_ours, x)
    ref.write_tensor(p_ref, x)
    assert open(p_ours, "rb").read() == open(p_ref, "rb").read()  # byte-identical containers
    assert nds.tensor_file_info(p_ref) == dims
    assert np.array_equal(nds.read_tensor(p_ref), x)
    assert np.array_equal(ref.read_tensor(p_ours), x)


def test_rejections(tmp_path):
    # tensor_file.cpp:67-96: magic, version, order, extents, truncated / trailing payload
    good = tmp_path / "g.ndt"
    nds.write_tensor(str(good), np.ones((2, 3), complex))
    raw = good.read_bytes()
    cases = {
        "magic": b"NDT2" + raw[4:],
        "version": raw[:4] + struct.pack("<I", 2) + raw[8:],
        "order": raw[:8] + struct.pack("<I", 0) + raw[12:],
        "extent": raw[:12] + struct.pack("<Q", 0) + raw[20:],
        "short": raw[:-8],
        "trailing": raw + b"\x00",
    }
    for name, blob in cases.items():
        p = tmp_path / f"{name}.ndt"
        p.write_bytes(blob)
        with pytest.raises(nds.TensorFileError):
            nds.read_tensor(str(p))
    with pytest.raises(nds.TensorFileError):
        nds.read_tensor(str(tmp_path / "missing.ndt"))
    with pytest.raises(nds.TensorFileError):
        nds.write_tensor(str(tmp_path / "no_such_dir" / "x.ndt"), np.ones(2, complex))


@pytest.mark.parametrize("dims,seed", [((2, 3), 401), ((3, 2, 2), 40), ((2, 2, 2, 2), 44)])
def test_random_ode_system_matches_reference(ref, dims, seed):
    a, f, x0 = nds.random_ode_system(dims, seed)
    ra, rf, rx0 = ref.random_ode_system(dims, seed)
    assert all(np.array_equal(m, r) for m, r in zip(a, ra))
    assert np.array_equal(f, rf) and np.array_equal(x0, rx0)
