import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: longer CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(params=["lane", "warp", "lane_noxs"])
def path(request, monkeypatch):
    """The evaluate paths: lane-per-chromosome (default when eligible), the
    general warp-per-chromosome kernel (FFS_DISABLE_LANE), and the lane path
    with the order kernel's unstaged variant (FFS_ORDER_NO_XS: machines read
    from global memory in pass D, the variant long rows take); both variables
    are read at state creation."""
    monkeypatch.delenv("FFS_DISABLE_LANE", raising=False)
    monkeypatch.delenv("FFS_ORDER_NO_XS", raising=False)
    if request.param == "warp":
        monkeypatch.setenv("FFS_DISABLE_LANE", "1")
    elif request.param == "lane_noxs":
        monkeypatch.setenv("FFS_ORDER_NO_XS", "1")
    return request.param
