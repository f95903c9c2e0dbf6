"""CPU checks of the boundary: the C-ABI library builds/loads and exports every
symbol include/ffs.h declares; the Python binding fails loudly without it."""
import ctypes
import os
import re

import pytest

from paper_1903_10741_b200 import build, ffs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "ffs.h")).read()
    return sorted(set(re.findall(r"FFS_API\s+[\w\s\*]*?\b(ffs_\w+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared() == sorted(ffs.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(build.build())
    for name in declared():
        assert hasattr(lib, name), name
    assert lib.ffs_version and ffs.lib().ffs_version().startswith(b"ffs-b200")


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.build()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_calls_fail_loudly():
    """Without a GPU every compute entry point reports an error, never a CPU result."""
    import numpy as np
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(ffs.FFSError) as e:
        ffs.Instance(1, 0, 1, 1, np.ones(1), np.ones(1), np.zeros(1), np.zeros(1), 1, 1)
    assert e.value.status == 4      # FFS_ERR_CUDA


def test_invalid_arguments_rejected_before_device():
    import numpy as np
    with pytest.raises(ffs.FFSError) as e:   # P must be > 0
        ffs.Instance(1, 0, 1, 1, np.zeros(1), np.ones(1), np.zeros(1), np.zeros(1), 1, 1)
    assert e.value.status == 1
    with pytest.raises(ffs.FFSError) as e:   # Q > Q_max
        ffs.Instance(1, 0, 1, 1, np.ones(1), np.full(1, 5), np.zeros(1), np.zeros(1), 1, 1)
    assert e.value.status == 2


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1903_10741_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                s = open(os.path.join(dp, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|ffs_oracle|or_ctx|or_decode)", s), f


def test_trace_csv_format(tmp_path):
    """RunTrace rows and CSV from a best record: best =
    trace_min, mean = trace_sum / population, one row per generation."""
    import numpy as np
    best = {"trace_min": np.array([30, 29, 29], np.int64), "trace_sum": np.array([100, 95, 90], np.int64)}
    rows = ffs.trace_rows(best, 4)
    assert rows == [(0, 30, 25.0), (1, 29, 23.75), (2, 29, 22.5)]
    p = tmp_path / "trace.csv"
    ffs.write_trace_csv(p, best, 4)
    assert p.read_text().splitlines() == ["generation,best_objective,mean_objective", "0,30,25.0", "1,29,23.75",
                                          "2,29,22.5"]
