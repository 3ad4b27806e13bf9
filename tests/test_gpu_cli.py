"""SURVEY 8(f)3 on the GPU: nds_random_problem vs the reference generator, multi-chunk NDT1
streaming to / from device memory, and the batch front end tools/cli/ndsylv_gpu (the reference
CLI's solve / ode / bench / selftest: output lines, CSV schema, exit codes)."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2412_15840_b200 as nds
from conftest import rel_max

pytestmark = pytest.mark.gpu
CLI = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "cli", "ndsylv_gpu")


def _cli(*args, timeout=300):
    if not os.path.exists(CLI):
        pytest.skip("tools/cli/ndsylv_gpu not built")
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("dims,seed", [((5, 4, 3), 905), ((2, 9, 33), 42), ((2,) * 8, 7)])
def test_random_problem_matches_reference(ctx, ref, dims, seed):
    a, x, b = ctx.random_problem(dims, seed)
    ra, rx, rb = ref.random_problem(list(dims), seed)
    assert all(np.array_equal(m, r) for m, r in zip(a, ra)) and np.array_equal(x, rx)
    assert rel_max(b, rb) <= 1e-14


def test_tensor_file_streaming_to_device(ctx, tmp_path):
    import torch
    dims = (256, 256, 160)  # 10.5 M entries = 168 MB: three pinned chunks each way
    total = int(np.prod(dims))
    x = torch.randn(total, dtype=torch.complex128, device="cuda")
    torch.cuda.synchronize()
    path = str(tmp_path / "big.ndt")
    ctx.write_tensor_dev(path, dims, x.data_ptr())
    assert os.path.getsize(path) == 12 + 8 * len(dims) + 16 * total
    y = torch.empty_like(x)
    ctx.read_tensor_dev(path, dims, y.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    host = nds.read_tensor(path)
    assert np.array_equal(host.ravel(order="F"), x.cpu().numpy())


def test_cli_solve_random_and_files(tmp_path):
    r = _cli("solve", "--random", "--dims", "5,4,3", "--seed", "7", "--out", str(tmp_path / "x.ndt"))
    assert r.returncode == 0, r.stderr
    err = float(re.search(r"max error vs known solution: (\S+)", r.stdout).group(1))
    res = float(re.search(r"residual: (\S+)", r.stdout).group(1))
    assert err <= 1e-9 and res <= 1e-9
    assert "dims: 5,4,3  (total 60)" in r.stdout and "timings: schur" in r.stdout
    # the same instance from files: coefficients + rhs written as NDT1, solved again
    ctx = nds.Context(0)
    a, x_true, b = ctx.random_problem((5, 4, 3), 7)
    paths = []
    for j, m in enumerate(a):
        paths.append(str(tmp_path / f"a{j}.ndt"))
        nds.write_tensor(paths[-1], m)
    nds.write_tensor(str(tmp_path / "b.ndt"), b)
    r2 = _cli("solve", "--coeffs", ",".join(paths), "--rhs", str(tmp_path / "b.ndt"), "--out", str(tmp_path / "x2.ndt"))
    assert r2.returncode == 0, r2.stderr
    assert rel_max(nds.read_tensor(str(tmp_path / "x2.ndt")), x_true) <= 1e-9
    assert np.array_equal(nds.read_tensor(str(tmp_path / "x.ndt")), nds.read_tensor(str(tmp_path / "x2.ndt")))


def test_cli_exit_codes(tmp_path):
    # ndsylv_main.cpp:366-381: 2 singular, 3 file, 4 memory budget, 1 other
    a1 = np.diag([1.0, -1.0]).astype(complex)
    a2 = np.diag([-1.0, 1.0]).astype(complex)
    nds.write_tensor(str(tmp_path / "a1.ndt"), a1)
    nds.write_tensor(str(tmp_path / "a2.ndt"), a2)
    nds.write_tensor(str(tmp_path / "b.ndt"), np.ones((2, 2), complex))
    coeffs = f"{tmp_path / 'a1.ndt'},{tmp_path / 'a2.ndt'}"
    assert _cli("solve", "--coeffs", coeffs, "--rhs", str(tmp_path / "b.ndt")).returncode == 2
    assert _cli("solve", "--coeffs", coeffs, "--rhs", str(tmp_path / "missing.ndt")).returncode == 3
    assert _cli("solve", "--random", "--dims", "64,64,64", "--max-mem", "1000").returncode == 4
    assert _cli("solve", "--bogus").returncode == 1
    assert _cli("ode", "--random", "--dims", "2,2").returncode == 1  # --t required


def test_cli_bench_csv_and_ode_and_selftest(tmp_path):
    csv = tmp_path / "bench.csv"
    r = _cli("bench", "--n-range", "2:12", "--seed", "3", "--csv", str(csv))
    assert r.returncode == 0, r.stderr
    lines = csv.read_text().splitlines()
    assert lines[0] == "# ndsylv bench csv 1"
    assert lines[1] == "N,total_size,schur_s,transform_s,backsub_s,inverse_s,total_s,max_error"
    rows = [l.split(",") for l in lines[2:]]
    assert [int(r_[0]) for r_ in rows] == list(range(2, 13))
    assert all(int(r_[1]) == 2 ** int(r_[0]) for r_ in rows)
    assert all(float(r_[7]) <= 1e-9 for r_ in rows)
    r = _cli("ode", "--random", "--dims", "2,3", "--seed", "401", "--t", "0.2", "--dt", "1e-3")
    assert r.returncode == 0, r.stderr
    assert float(re.search(r"max discrepancy: (\S+)", r.stdout).group(1)) <= 1e-8
    r = _cli("selftest")
    assert r.returncode == 0 and "selftest: all ok" in r.stdout, r.stdout + r.stderr
