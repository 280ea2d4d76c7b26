"""The C ABI library loads and exports every symbol include/ebem_gpu.h declares;
without a GPU every compute entry fails loudly (no CPU fallback).  CPU only."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "ebem_gpu.h"
SO = ROOT / "paper_2411_18026_b200" / "libebem_gpu.so"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ebem_gpu_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ["ebem_gpu_problem_create", "ebem_gpu_true_block", "ebem_gpu_cell_basis",
                 "ebem_gpu_fds_create", "ebem_gpu_fds_solve", "ebem_gpu_fds_rank_of",
                 "ebem_gpu_rhs_plane", "ebem_gpu_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    assert SO.exists(), "build with __graft_entry__.build()"
    lib = ctypes.CDLL(str(SO))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def _has_gpu():
    lib = ctypes.CDLL(str(SO))
    buf = ctypes.create_string_buffer(128)
    return lib.ebem_gpu_device_info(buf, 128) == 0


def test_no_gpu_fails_loudly(eb):
    if _has_gpu():
        pytest.skip("a GPU is present")
    mesh = eb.Mesh.star(64, eb.StarShape(1.0, 0.0, 3))
    med = eb.Medium.from_lame(1.0, 1.0, 1.0, 1.0)
    with pytest.raises(eb.CudaError):
        eb.BlockAssembler(mesh, med, med.default_coupling())
    with pytest.raises(eb.CudaError):
        eb.eval_hankel([1.0])
