"""TEST INFRASTRUCTURE: numpy/ctypes bindings of the two CPU checkers.

  ORC  oracle/liboracle.so            plain-C restatement (oracle/hpclust_oracle.c)
  REF  oracle/_ref/libhpclust_ref.so  the reference headers compiled in place (may be absent)
Both expose the same calling conventions so tests can pin ORC against REF.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
P, I64, I32, U64, D, SZ = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_double, C.c_size_t


def ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p).value


class RunCfg(C.Structure):
    _fields_ = [("k", U64), ("sample_size", U64), ("n_workers", U64), ("max_samples", U64), ("time_limit", D),
                ("strategy", I32), ("phase_t1", D), ("phase_t2", D), ("master_seed", U64), ("candidates", U64),
                ("max_iters", U64), ("rel_tol", D), ("n_threads", U64), ("compute_full_objective", I32),
                ("compute_assignment", I32)]


class RunOut(C.Structure):
    _fields_ = [("full_objective", D), ("has_full_objective", I32), ("best_worker", I32),
                ("best_sample_objective", D), ("clustering_time", D), ("clustering_time_first_finisher", D),
                ("wall_seconds", D), ("total_samples", U64), ("distance_evals", I64), ("n_publications", I64)]


class CheckerError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class _Checker:
    prefix = ""

    def __init__(self, path):
        self.lib = C.CDLL(str(path))
        self.path = path

    def _err(self, rc):
        if rc:
            raise CheckerError(rc, getattr(self.lib, self.prefix + "last_error")().decode())


class Oracle(_Checker):
    """The C restatement."""

    prefix = "orc_"

    def __init__(self, path=ROOT / "oracle" / "liboracle.so"):
        super().__init__(path)
        L = self.lib
        L.orc_last_error.restype = C.c_char_p
        L.orc_sizeof_rng.restype = SZ
        L.orc_rng_next_u64.restype = U64
        L.orc_rng_next_unit.restype = D
        L.orc_rng_uniform_index.restype = U64
        L.orc_rng_uniform_index.argtypes = [P, U64]
        L.orc_rng_seed.argtypes = [P, U64]
        L.orc_rng_derive.argtypes = [P, U64, U64, U64]
        L.orc_rng_next_u64.argtypes = [P]
        L.orc_rng_next_unit.argtypes = [P]
        L.orc_splitmix64.restype = U64
        L.orc_splitmix64.argtypes = [U64]
        L.orc_assign.argtypes = [P, SZ, SZ, P, P, SZ, SZ, P, P, P, P]
        L.orc_kmeans.argtypes = [P, SZ, SZ, P, P, SZ, SZ, D, SZ, P, P, P, P, P, P, P, P, P, I64, P]
        L.orc_reinit_degenerate.argtypes = [P, SZ, SZ, P, P, SZ, SZ, SZ, P, P, P, P]
        L.orc_seed_with_uniforms.argtypes = [P, SZ, SZ, P, P, SZ, SZ, SZ, P, P, P, P, P]
        L.orc_draw_indices.argtypes = [SZ, SZ, P, P]
        L.orc_run.argtypes = [P, SZ, SZ, P, P, P, P, P, P, I64, P, P, I64, P]
        self.rng_size = L.orc_sizeof_rng()

    def rng(self, seed=None, derive=None):
        buf = C.create_string_buffer(self.rng_size)
        if derive is not None:
            self.lib.orc_rng_derive(buf, *[C.c_uint64(v) for v in derive])
        else:
            self.lib.orc_rng_seed(buf, C.c_uint64(seed))
        return buf

    def next_u64(self, r):
        return self.lib.orc_rng_next_u64(r)

    def next_unit(self, r):
        return self.lib.orc_rng_next_unit(r)

    def uniform_index(self, r, n):
        return self.lib.orc_rng_uniform_index(r, n)

    def assign(self, X, C_, flags=None, n_chunks=1):
        X = np.ascontiguousarray(X, np.float64)
        C_ = np.ascontiguousarray(C_, np.float64)
        m, n = X.shape
        k = C_.shape[0]
        labels = np.empty(m, np.int32)
        counts = np.empty(k, np.int64)
        cost = C.c_double()
        nd = C.c_int64()
        fl = None if flags is None else np.ascontiguousarray(flags, np.uint8)
        self._err(self.lib.orc_assign(ptr(X), m, n, ptr(C_), ptr(fl), k, n_chunks, ptr(labels), ptr(counts),
                                      C.byref(cost), C.byref(nd)))
        return labels, counts, cost.value, nd.value

    def kmeans(self, S, C0, max_iters=300, rel_tol=1e-4, n_chunks=1, flags=None):
        S = np.ascontiguousarray(S, np.float64)
        C0 = np.ascontiguousarray(C0, np.float64)
        s, n = S.shape
        k = C0.shape[0]
        Co = np.empty((k, n))
        fo = np.empty(k, np.uint8)
        lab = np.empty(s, np.int32)
        cnt = np.empty(k, np.int64)
        obj = C.c_double()
        it = C.c_int64()
        st = C.c_int32()
        nd = C.c_int64()
        cap = max_iters + 2
        hist = np.empty(cap)
        hl = C.c_int64()
        fl = None if flags is None else np.ascontiguousarray(flags, np.uint8)
        self._err(self.lib.orc_kmeans(ptr(S), s, n, ptr(C0), ptr(fl), k, max_iters, rel_tol, n_chunks, ptr(Co),
                                      ptr(fo), ptr(lab), ptr(cnt), C.byref(obj), C.byref(it), C.byref(st),
                                      C.byref(nd), ptr(hist), cap, C.byref(hl)))
        return dict(centroids=Co, degenerate=fo, labels=lab, counts=cnt, objective=obj.value,
                    iterations=it.value, stop=st.value, n_d=nd.value, history=hist[: hl.value].copy())

    def reinit(self, S, C0, flags, rng, candidates=3):
        S = np.ascontiguousarray(S, np.float64)
        C0 = np.ascontiguousarray(C0, np.float64)
        s, n = S.shape
        k = C0.shape[0]
        Co = np.empty((k, n))
        fo = np.empty(k, np.uint8)
        nd = C.c_int64()
        fl = np.ascontiguousarray(flags, np.uint8)
        self._err(self.lib.orc_reinit_degenerate(ptr(S), s, n, ptr(C0), ptr(fl), k, candidates, 1, rng, ptr(Co),
                                                 ptr(fo), C.byref(nd)))
        return Co, fo, nd.value

    def seed_with_uniforms(self, S, C0, flags, first_row, units, candidates=3):
        S = np.ascontiguousarray(S, np.float64)
        C0 = np.ascontiguousarray(C0, np.float64)
        s, n = S.shape
        k = C0.shape[0]
        Co = np.empty((k, n))
        fo = np.empty(k, np.uint8)
        nd = C.c_int64()
        filled = C.c_int64()
        un = np.ascontiguousarray(units, np.float64)
        fl = np.ascontiguousarray(flags, np.uint8)
        self._err(self.lib.orc_seed_with_uniforms(ptr(S), s, n, ptr(C0), ptr(fl), k, candidates, first_row,
                                                  ptr(un), ptr(Co), ptr(fo), C.byref(nd), C.byref(filled)))
        return Co, fo, nd.value, filled.value

    def draw_indices(self, m, s, rng):
        out = np.empty(s, np.int64)
        self._err(self.lib.orc_draw_indices(m, s, rng, ptr(out)))
        return out

    def run(self, X, **kw):
        return _run(self, "orc_run", X, **kw)


class Reference(_Checker):
    """The reference headers compiled in place (oracle/_ref)."""

    prefix = "hpref_"

    def __init__(self, path=ROOT / "oracle" / "_ref" / "libhpclust_ref.so"):
        super().__init__(path)
        L = self.lib
        L.hpref_last_error.restype = C.c_char_p
        L.hpref_rng_new.restype = P
        L.hpref_rng_new.argtypes = [U64]
        L.hpref_rng_derive.restype = P
        L.hpref_rng_derive.argtypes = [U64, U64, U64]
        L.hpref_rng_clone.restype = P
        L.hpref_rng_clone.argtypes = [P]
        L.hpref_rng_free.argtypes = [P]
        L.hpref_rng_next_u64.restype = U64
        L.hpref_rng_next_u64.argtypes = [P]
        L.hpref_rng_next_unit.restype = D
        L.hpref_rng_next_unit.argtypes = [P]
        L.hpref_rng_uniform_index.restype = U64
        L.hpref_rng_uniform_index.argtypes = [P, U64]
        L.hpref_splitmix64.restype = U64
        L.hpref_splitmix64.argtypes = [U64]
        L.hpref_assign.argtypes = [P, SZ, SZ, P, P, SZ, SZ, P, P, P, P]
        L.hpref_mssc_objective.argtypes = [P, SZ, SZ, P, SZ, SZ, P]
        L.hpref_kmeans.argtypes = [P, SZ, SZ, P, P, SZ, SZ, D, P, P, P, P, P, P, P, P, P, I64, P]
        L.hpref_reinit_degenerate.argtypes = [P, SZ, SZ, P, P, SZ, SZ, P, P, P, P]
        L.hpref_draw_indices.argtypes = [SZ, SZ, P, P]
        L.hpref_draw_sample.argtypes = [P, SZ, SZ, SZ, P, P]
        L.hpref_run.argtypes = [P, SZ, SZ, P, P, P, P, P, P, I64, P, P, I64, P]
        L.hpref_gen_blobs.argtypes = [SZ, SZ, SZ, D, D, D, D, SZ, D, D, U64, P]
        L.hpref_brute_force.argtypes = [P, SZ, SZ, SZ, P, P, P]
        L.hpref_kmeans_threads.argtypes = [P, SZ, SZ, SZ, P, SZ, SZ, D, P, P]
        if hasattr(L, "hpref_baseline"):
            L.hpref_baseline.argtypes = [P, SZ, SZ, SZ, SZ, U64, SZ, D, P, P, P, P, P, P]

    def baseline(self, X, k, p, seed, max_iters=300, rel_tol=1e-4):
        """baselines.hpp forgy_kmeans (p = 0) / pbk_bdc (segment size p) with RngStream(seed)."""
        X = np.ascontiguousarray(X, np.float64)
        m, n = X.shape
        Co = np.empty((k, n))
        fo = np.empty(k, np.uint8)
        lab = np.empty(m, np.int32)
        f, nd, samples = D(), C.c_int64(), C.c_int64()
        self._err(self.lib.hpref_baseline(ptr(X), m, n, k, p, seed, max_iters, rel_tol, ptr(Co), ptr(fo), ptr(lab),
                                          C.byref(f), C.byref(nd), C.byref(samples)))
        return dict(centroids=Co, degenerate=fo, labels=lab, full_objective=f.value, n_d=nd.value,
                    total_samples=samples.value)

    def rng(self, seed=None, derive=None):
        h = self.lib.hpref_rng_derive(*derive) if derive is not None else self.lib.hpref_rng_new(seed)
        return _RefRng(self.lib, h)

    def assign(self, X, C_, flags=None, n_chunks=1):
        X = np.ascontiguousarray(X, np.float64)
        C_ = np.ascontiguousarray(C_, np.float64)
        m, n = X.shape
        k = C_.shape[0]
        labels = np.empty(m, np.int32)
        counts = np.empty(k, np.int64)
        cost = C.c_double()
        nd = C.c_int64()
        fl = None if flags is None else np.ascontiguousarray(flags, np.uint8)
        self._err(self.lib.hpref_assign(ptr(X), m, n, ptr(C_), ptr(fl), k, n_chunks, ptr(labels), ptr(counts),
                                        C.byref(cost), C.byref(nd)))
        return labels, counts, cost.value, nd.value

    def kmeans(self, S, C0, max_iters=300, rel_tol=1e-4, flags=None):
        S = np.ascontiguousarray(S, np.float64)
        C0 = np.ascontiguousarray(C0, np.float64)
        s, n = S.shape
        k = C0.shape[0]
        Co = np.empty((k, n))
        fo = np.empty(k, np.uint8)
        lab = np.empty(s, np.int32)
        cnt = np.empty(k, np.int64)
        obj = C.c_double()
        it = C.c_int64()
        st = C.c_int32()
        nd = C.c_int64()
        cap = max_iters + 2
        hist = np.empty(cap)
        hl = C.c_int64()
        fl = None if flags is None else np.ascontiguousarray(flags, np.uint8)
        self._err(self.lib.hpref_kmeans(ptr(S), s, n, ptr(C0), ptr(fl), k, max_iters, rel_tol, ptr(Co), ptr(fo),
                                        ptr(lab), ptr(cnt), C.byref(obj), C.byref(it), C.byref(st), C.byref(nd),
                                        ptr(hist), cap, C.byref(hl)))
        return dict(centroids=Co, degenerate=fo, labels=lab, counts=cnt, objective=obj.value,
                    iterations=it.value, stop=st.value, n_d=nd.value, history=hist[: hl.value].copy())

    def reinit(self, S, C0, flags, rng, candidates=3):
        S = np.ascontiguousarray(S, np.float64)
        C0 = np.ascontiguousarray(C0, np.float64)
        s, n = S.shape
        k = C0.shape[0]
        Co = np.empty((k, n))
        fo = np.empty(k, np.uint8)
        nd = C.c_int64()
        fl = np.ascontiguousarray(flags, np.uint8)
        self._err(self.lib.hpref_reinit_degenerate(ptr(S), s, n, ptr(C0), ptr(fl), k, candidates, rng.h, ptr(Co),
                                                   ptr(fo), C.byref(nd)))
        return Co, fo, nd.value

    def draw_indices(self, m, s, rng):
        out = np.empty(s, np.int64)
        self._err(self.lib.hpref_draw_indices(m, s, rng.h, ptr(out)))
        return out

    def gen_blobs(self, num_points, features, num_blobs, center=(-40.0, 40.0), std=(0.0, 10.0), noise_points=500,
                  noise=(-50.0, 50.0), seed=0):
        X = np.empty((num_points + noise_points, features))
        self._err(self.lib.hpref_gen_blobs(num_points, features, num_blobs, center[0], center[1], std[0], std[1],
                                           noise_points, noise[0], noise[1], C.c_uint64(seed), ptr(X)))
        return X

    def brute_force(self, X, k):
        X = np.ascontiguousarray(X, np.float64)
        m, n = X.shape
        Co = np.empty((k, n))
        fo = np.empty(k, np.uint8)
        cost = C.c_double()
        self._err(self.lib.hpref_brute_force(ptr(X), m, n, k, ptr(Co), ptr(fo), C.byref(cost)))
        return Co, fo, cost.value

    def kmeans_threads(self, samples, inits, max_iters=300, rel_tol=1e-4):
        samples = np.ascontiguousarray(samples, np.float64)
        inits = np.ascontiguousarray(inits, np.float64)
        W, s, n = samples.shape
        k = inits.shape[1]
        nd = C.c_int64()
        obj = np.empty(W)
        self._err(self.lib.hpref_kmeans_threads(ptr(samples), W, s, n, ptr(inits), k, max_iters, rel_tol,
                                                C.byref(nd), ptr(obj)))
        return nd.value, obj

    def run(self, X, **kw):
        return _run(self, "hpref_run", X, **kw)


class _RefRng:
    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def next_u64(self):
        return self.lib.hpref_rng_next_u64(self.h)

    def next_unit(self):
        return self.lib.hpref_rng_next_unit(self.h)

    def uniform_index(self, n):
        return self.lib.hpref_rng_uniform_index(self.h, n)

    def clone(self):
        return _RefRng(self.lib, self.lib.hpref_rng_clone(self.h))

    def __del__(self):
        try:
            self.lib.hpref_rng_free(self.h)
        except Exception:
            pass


STRATS = {"inner": 0, "competitive": 1, "cooperative": 2, "collective": 2, "hybrid": 3}


def _run(chk, fname, X, *, k, sample_size, n_workers, max_samples, strategy="competitive", t1=0.0, t2=0.0, seed=0,
         candidates=3, max_iters=300, rel_tol=1e-4, n_threads=4, full=True, assignment=False):
    X = np.ascontiguousarray(X, np.float64)
    m, n = X.shape
    cfg = RunCfg(k, sample_size, n_workers, max_samples, -1.0, STRATS[strategy], t1, t2, seed, candidates, max_iters,
                 rel_tol, n_threads, int(full), int(assignment))
    o = RunOut()
    W = 1 if strategy == "inner" else n_workers
    cent = np.empty((k, n))
    flags = np.empty(k, np.uint8)
    labels = np.empty(m, np.int32) if assignment else None
    pub_cap = max(64, max_samples * W)
    pubs = np.zeros((pub_cap, 4))
    wobj = np.empty(W)
    tcap = max_samples
    traces = np.zeros((W, tcap, 2))
    tlen = np.zeros(W, np.int64)
    rc = getattr(chk.lib, fname)(ptr(X), m, n, C.byref(cfg), C.byref(o), ptr(cent), ptr(flags), ptr(labels),
                                 ptr(pubs), pub_cap, ptr(wobj), ptr(traces), tcap, ptr(tlen))
    chk._err(rc)
    return dict(centroids=cent, degenerate=flags, labels=labels, full_objective=o.full_objective,
                has_full_objective=o.has_full_objective, best_worker=o.best_worker,
                best_sample_objective=o.best_sample_objective, clustering_time=o.clustering_time,
                clustering_time_first_finisher=o.clustering_time_first_finisher, total_samples=o.total_samples,
                distance_evals=o.distance_evals, publications=pubs[: o.n_publications].copy(), worker_obj=wobj,
                traces=[traces[w, : tlen[w]].copy() for w in range(W)])


class RefInject:
    """oracle/_ref/libhpclust_ref_inject.so: the reference's own worker step (reinit_degenerate +
    kmeans, engine.hpp:238-267) with injected 64-bit random draws (oracle/ref_inject.cpp)."""

    def __init__(self, path):
        self.lib = L = C.CDLL(str(path))
        P, SZ, I64, D = C.c_void_p, C.c_size_t, C.c_int64, C.c_double
        L.hpref_inject_last_error.restype = C.c_char_p
        L.hpref_inject_step.argtypes = [P, SZ, SZ, P, P, SZ, SZ, SZ, D, P, I64, P, P, P, P, P, P, P, P, P]

    @staticmethod
    def philox_draws(first_row, units, no_valid):
        """The u64 draws that make the reference consume first_row (uniform_index, rng.hpp:43-53:
        x < limit, x % s) and the given units (next_unit, rng.hpp:38-40: (v >> 11) * 2^-53)."""
        v = [int(first_row)] if no_valid else []
        v += [int(round(u * 2.0 ** 53)) << 11 for u in np.asarray(units, np.float64)]
        return np.array(v, dtype=np.uint64)

    def step(self, S, C0, flags, draws, candidates=3, max_iters=300, rel_tol=1e-4, labels=False):
        S = np.ascontiguousarray(S, np.float64)
        s, n = S.shape
        C0 = np.ascontiguousarray(C0, np.float64)
        k = C0.shape[0]
        fl = np.ascontiguousarray(flags, np.uint8)
        draws = np.ascontiguousarray(draws, np.uint64)
        Cs, Co, fo = np.empty((k, n)), np.empty((k, n)), np.empty(k, np.uint8)
        f, it, st, nd, used = C.c_double(), C.c_int64(), C.c_int32(), C.c_int64(), C.c_int64()
        lab = np.empty(s, np.int32) if labels else None
        rc = self.lib.hpref_inject_step(ptr(S), s, n, ptr(C0), ptr(fl), k, candidates, max_iters, rel_tol,
                                        ptr(draws), len(draws), ptr(Cs), ptr(Co), ptr(fo), C.byref(f), C.byref(it),
                                        C.byref(st), C.byref(nd), C.byref(used), ptr(lab))
        if rc != 0:
            raise RuntimeError(self.lib.hpref_inject_last_error().decode())
        return dict(seeded=Cs, centroids=Co, degenerate=fo, objective=f.value, iterations=it.value, stop=st.value,
                    n_d=nd.value, consumed=used.value, labels=lab)


_ORC = _REF = _INJ = None


def ref_inject() -> RefInject | None:
    global _INJ
    p = ROOT / "oracle" / "_ref" / "libhpclust_ref_inject.so"
    if _INJ is None and p.exists():
        _INJ = RefInject(p)
    return _INJ


def orc() -> Oracle:
    global _ORC
    if _ORC is None:
        _ORC = Oracle()
    return _ORC


def ref() -> Reference | None:
    global _REF
    p = ROOT / "oracle" / "_ref" / "libhpclust_ref.so"
    if _REF is None and p.exists():
        _REF = Reference(p)
    return _REF


def chunk_range_py(rows: int, n_chunks: int, chunk: int):
    """parallel.hpp:106-112 chunk_range: the rows of part `chunk` of `n_chunks` (the first rows % n_chunks
    parts get one extra row) -- the row shard of rank `chunk` in a multi-GPU run."""
    base, extra = divmod(rows, n_chunks)
    b = chunk * base + min(chunk, extra)
    return b, b + base + (1 if chunk < extra else 0)
