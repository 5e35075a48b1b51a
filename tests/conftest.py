import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size (BASELINE.json) cases")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def kats():
    return load_golden("kats.json")


@pytest.fixture(scope="session")
def seeded_cases():
    return load_golden("seeded_cases.json")


@pytest.fixture(scope="session")
def acceptance_cases():
    return load_golden("acceptance_1000.json")


@pytest.fixture(scope="session")
def quant_cases():
    return load_golden("quant.json")


@pytest.fixture(scope="session")
def large_cases():
    p = os.path.join(GOLDEN, "large.json")
    if not os.path.exists(p):
        pytest.skip("large.json golden not generated")
    return load_golden("large.json")


@pytest.fixture(scope="session")
def cuda_lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2406_11674_b200 import _lib
    return _lib.lib()


def gemv_check(y, W, x, tol=1e-3):
    """North star GEMV tolerance, element-wise:
    every row r satisfies |y_r - y_ref_r| <= tol * sum_j |W_rj x_j| (the
    conditioning of that dot product), and rows whose |y_ref_r| is not
    dominated by cancellation (|y_ref_r| >= 0.01 sum_j |W_rj x_j|; a random
    row of length n sits near 1.25/sqrt(n) of that sum, so at the catalog
    widths most rows qualify) also satisfy
    the plain relative bound |y_r - y_ref_r| <= tol * |y_ref_r|.  y_ref is the
    float64 product over the same f16 W and x.  Returns (max error/mag,
    max relative error over well-conditioned rows)."""
    import torch
    y = y.detach().double().cpu().reshape(-1)
    Wd = W.detach().cpu().double()
    xd = x.detach().cpu().double().reshape(-1)
    ref = Wd @ xd
    mag = Wd.abs() @ xd.abs()
    err = (y - ref).abs()
    finite = torch.isfinite(ref)
    assert torch.equal(torch.isfinite(y), finite), "non-finite pattern differs from the reference"
    err, ref, mag = err[finite], ref[finite], mag[finite]
    bound = tol * mag + 1e-30
    bad = err > bound
    assert not bad.any(), f"{int(bad.sum())} rows exceed {tol} * sum|W x|; worst {float((err / bound).max())}"
    good = (ref.abs() >= 0.01 * mag) & (mag > 0)
    rel = (err[good] / ref[good].abs()).max().item() if good.any() else 0.0
    assert rel <= tol, f"per-element relative error {rel} > {tol}"
    return float((err / (mag + 1e-30)).max()) if err.numel() else 0.0, rel


def gemm_check(y, W, X, tol=1e-3):
    """gemv_check for Y = X W^T ([tokens, rows]), element-wise, in float64 on
    Y's device: |Y_tr - ref_tr| <= tol * sum_j |X_tj W_rj| everywhere, and
    <= tol * |ref_tr| where ref_tr is not dominated by cancellation.  Returns
    (max error/mag, max relative error over well-conditioned entries)."""
    import torch
    dev = y.device
    Wd = W.to(dev).double()
    Xd = X.to(dev).double()
    ref = Xd @ Wd.T
    mag = Xd.abs() @ Wd.abs().T
    yd = y.double()
    assert yd.shape == ref.shape, (yd.shape, ref.shape)
    err = (yd - ref).abs()
    bound = tol * mag + 1e-30
    bad = err > bound
    assert not bad.any(), f"{int(bad.sum())} entries exceed {tol} * sum|X W|; worst {float((err / bound).max())}"
    good = (ref.abs() >= 0.01 * mag) & (mag > 0)
    rel = (err[good] / ref[good].abs()).max().item() if good.any() else 0.0
    assert rel <= tol, f"per-element relative error {rel} > {tol}"
    return float((err / (mag + 1e-30)).max()) if err.numel() else 0.0, rel
