"""CPU: the C-ABI library loads, exports exactly what include/hpcg.h declares, fails loudly
without a GPU (no CPU fallback), and its host-side reference-stream replay (the only host
computation in the product: RNG draws for parity mode) is bit-identical to the reference."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2311_04517_b200 as hp
from paper_2311_04517_b200 import _lib
from oracle_py import orc, ref

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "hpcg.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(hpcg_\w+)\s*\(", text, re.M)))


def test_header_declares_what_the_binding_binds():
    assert set(declared_symbols()) == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.hpcg_abi_version() == 2  # hpcg.h HPCG_ABI_VERSION (the binding checks it at load)


def test_library_is_sm100a_cuda_code():
    data = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in data  # fatbin compiled for sm_100a only


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(hp.CudaError):
        hp.Context(0)
    with pytest.raises(hp.CudaError):
        hp.mssc_objective(np.zeros((1, 2)), np.zeros((3, 2)))


@pytest.mark.parametrize("seed", [0, 1, 12345, 2**63 + 7])
def test_reference_stream_replay_matches_reference(seed):
    a = hp.RngStream(seed)
    o = orc()
    b = o.rng(seed=seed)
    for _ in range(700):  # crosses the 312-word twist boundary twice
        assert a.next_u64() == o.next_u64(b)
    for n in (1, 7, 1000003, 2**40 + 3):
        assert a.uniform_index(n) == o.uniform_index(b, n)
    assert a.next_unit() == o.next_unit(b)
    R = ref()
    if R is not None:
        c = R.rng(seed=seed)
        d = hp.RngStream(seed)
        for _ in range(50):
            assert d.next_u64() == c.next_u64()


def test_derived_streams_and_sparse_fisher_yates():
    # engine.hpp:457 stream derivation + engine.hpp:165-177 draw order, in O(s)
    o = orc()
    for (m, s, master, wi) in [(1000, 50, 0, 0), (5000, 400, 7, 3), (64, 64, 1, 1), (10**9, 2000, 3, 5)]:
        a = hp.RngStream.derive(master, 1, wi)
        idx = hp.reference_draw_indices(m, s, a)
        assert len(set(idx.tolist())) == s and idx.min() >= 0 and idx.max() < m
        if m <= 10**6:
            b = o.rng(derive=(master, 1, wi))
            assert np.array_equal(idx, o.draw_indices(m, s, b))
            assert a.next_u64() == o.next_u64(b)


def test_argument_validation_errors_are_reference_texts():
    with pytest.raises(hp.InvalidArgument, match="kmeans: max_iters must be positive"):
        hp.kmeans(np.zeros((3, 1)), np.zeros((1, 1)), hp.LloydConfig(max_iters=0))
    with pytest.raises(hp.InvalidArgument, match="kmeans: rel_tol must be positive"):
        hp.kmeans(np.zeros((3, 1)), np.zeros((1, 1)), hp.LloydConfig(rel_tol=0.0))
    with pytest.raises(hp.InvalidArgument, match="kmeans: degenerate centroid in init"):
        hp.kmeans(np.zeros((3, 1)), np.zeros((1, 1)), degenerate=np.ones(1, np.uint8))
    with pytest.raises(hp.InvalidArgument, match="assign_nearest: degenerate centroid present"):
        hp.assign_nearest(np.zeros((3, 1)), np.zeros((1, 1)), degenerate=np.ones(1, np.uint8))
    with pytest.raises(hp.InvalidArgument, match="draw_sample: sample size must be in"):
        hp.reference_draw_indices(5, 6, hp.RngStream(1))
    with pytest.raises(hp.NoSolutionError):
        hp.select_best([float("inf")] * 3)
    assert hp.select_best([5.0, 3.0, 9.0]) == 1 and hp.select_best([3.0, 3.0]) == 0
