"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every entry point include/*.h declares (no device calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rdmm_[a-z0-9_]+)\s*\(", src)))


def exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True,
                         text=True, check=True).stdout
    return {ln.split()[-1] for ln in out.splitlines() if " T " in ln}


def test_cuda_capi_exports_every_declared_symbol():
    import paper_2311_18141_b200._lib as L

    names = declared("rdmm_cuda.h")
    assert len(names) >= 10
    syms = exported(L.LIB_PATH)
    missing = [n for n in names if n not in syms]
    assert not missing, missing
    lib = ctypes.CDLL(L.LIB_PATH)
    for n in names:
        assert hasattr(lib, n)


def test_host_capi_exports_every_declared_symbol():
    import paper_2311_18141_b200._lib as L

    names = declared("rdmm_host.h")
    assert "rdmm_h_run_multiply" in names
    syms = exported(L.LIB_PATH)
    assert not [n for n in names if n not in syms]


def test_fabric_capi_declared():
    names = declared("rdmm_cuda.h")
    for n in ("rdmm_fabric_create", "rdmm_get_nb", "rdmm_wait", "rdmm_fetch_add_i64",
              "rdmm_queue_push", "rdmm_queue_pop", "rdmm_barrier", "rdmm_heap_alloc",
              "rdmm_spgemm_symbolic", "rdmm_spgemm_numeric", "rdmm_spmm_csr_f32"):
        assert n in names


def test_error_taxonomy_mapping():
    import paper_2311_18141_b200 as rd

    assert issubclass(rd.HeapExhaustedError, rd.FabricError)
    assert issubclass(rd.QueueFullError, rd.FabricError)
    assert issubclass(rd.ProtocolError, rd.FabricError)
    assert rd._lib.rdmm_version().startswith(b"rdmm-b200")


def test_library_is_sm100a_only():
    import paper_2311_18141_b200._lib as L

    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True,
                         text=True).stdout
    if not out:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_host_permutation_matches_reference(golden, orc):
    """rdmm_permutation (host part of permute_symmetric, gen.hpp:141-147):
    relabelling rmat(8, 8, seed=1) with it reproduces the reference golden."""
    import numpy as np

    from paper_2311_18141_b200.tile import permutation

    a = orc.rmat(8, 8, seed=1)
    perm = permutation(a.rows, 5).astype(np.int64)
    assert np.array_equal(np.sort(perm), np.arange(a.rows))
    r = np.repeat(np.arange(a.rows), np.diff(a.row_ptr.astype(np.int64)))
    nr, nc = perm[r], perm[a.col_idx.astype(np.int64)]
    order = np.lexsort((nc, nr))
    rp = np.concatenate([[0], np.cumsum(np.bincount(nr, minlength=a.rows))])
    assert np.array_equal(rp, golden["perm8_rp"])
    assert np.array_equal(nc[order], golden["perm8_ci"])
    assert np.array_equal(a.values[order], golden["perm8_v"])
