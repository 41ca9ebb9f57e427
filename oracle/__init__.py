"""BFLA CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2605_12193_b200``) never imports it and shares no code with it.

Thin ctypes wrapper over ``bfla_oracle.c`` (plain C, fp64 attention, canonical fp32 mask
arithmetic).  Each wrapper names the paper passage of the C function it calls; see the C file
for the step-by-step definitions and DESIGN.md §3-4 for the readings.

Parity status: every function below is pinned by ``tests/test_oracle_*.py`` except the
paper-level densities of Tab.mask (need LongBench + model weights) — "parity unpinned" for
those end-to-end numbers only.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bfla_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

POOL_FLATTEN, POOL_MEAN = 0, 1
SELECT_MASS, SELECT_RATIO = 0, 1
LBL_DROP, LBL_MASS, LBL_SINK, LBL_BAND, LBL_STRIDE, LBL_RANDOM = range(6)

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, -O2 -ffp-contract=off -mfma -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-mfma", "-fopenmp", "-fPIC",
                               "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I, F, D, U64 = ctypes.c_int, ctypes.c_float, ctypes.c_double, ctypes.c_uint64
        lib.orc_causal.argtypes = [I, I, I, I, I]
        lib.orc_causal.restype = I
        lib.orc_flatten.argtypes = [P, I, I, I, I, I, P, P]
        lib.orc_block_scores.argtypes = [P, P, I, I, I, I, I, I, I, I, P]
        lib.orc_exp2_canon.argtypes = [F]
        lib.orc_exp2_canon.restype = F
        lib.orc_block_softmax_row.argtypes = [P, I, I, P]
        lib.orc_keep_select.argtypes = [P, P, I, I, F, F, P, P, P, P, P]
        lib.orc_keep_select.restype = I
        lib.orc_select.argtypes = [P, I, I, I, I, I, I, I, F, F, P, P, P, P, P, P, P, P]
        lib.orc_mix64.argtypes = [U64]
        lib.orc_mix64.restype = U64
        lib.orc_chi.argtypes = [I, I, U64]
        lib.orc_chi.restype = U64
        lib.orc_psi.argtypes = [I, I, I, U64]
        lib.orc_psi.restype = D
        lib.orc_expand_rescue.argtypes = [P, I, I, I, I, I, I, I, I, D, U64, I, P]
        lib.orc_masked_attention.argtypes = [P, P, P, I, I, I, I, I, D, P, I, I, P, P, P, P]
        lib.orc_causal_tiles.argtypes = [I, I, I]
        lib.orc_causal_tiles.restype = ctypes.c_long
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def cdiv(a: int, b: int) -> int:
    return -(-a // b)


# ---------------------------------------------------------------- Eq. 11-13
def causal(i: int, j: int, blk: int, n_q: int, n_kv: int) -> bool:
    """Eq. 11-13: block (i, j) is causal iff j*blk <= min(N_c + (i+1)*blk - 1, N_kv - 1)."""
    return bool(_L().orc_causal(i, j, blk, n_q, n_kv))


def causal_tiles(n_q: int, n_kv: int, T: int) -> int:
    """Number of causal (i, j) tiles at tile size T (kappa denominator, R20)."""
    return int(_L().orc_causal_tiles(n_q, n_kv, T))


# ---------------------------------------------------------------- Eq. 4-7
def flatten(x, b: int, g: int):
    """Eq. 4-7: Phi(X) [H, L, G, g*C] and valid-group flags [L, G] (R2, R3)."""
    x = _f32(x)
    H, N, C = x.shape
    L, G = cdiv(N, b), b // g
    out = np.empty((H, L, G, g * C), np.float32)
    valid = np.empty((L, G), np.uint8)
    _L().orc_flatten(_p(x), H, N, C, b, g, _p(out), _p(valid))
    return out, valid


# ---------------------------------------------------------------- Eq. 9-10, 14
def block_scores(q, k, b: int, g: int, pool: int = POOL_FLATTEN) -> np.ndarray:
    """Eq. 9-10 (+ Eq. 14): S [Hq, Lq, Lkv] fp32, -inf on non-causal blocks.

    q: [Hq, Nq, C], k: [Hkv, Nkv, C] — fp32 arrays holding the bf16 inputs exactly.
    """
    q, k = _f32(q), _f32(k)
    Hq, Nq, C = q.shape
    Hkv, Nkv, _ = k.shape
    S = np.empty((Hq, cdiv(Nq, b), cdiv(Nkv, b)), np.float32)
    _L().orc_block_scores(_p(q), _p(k), Hq, Hkv, Nq, Nkv, C, b, g, pool, _p(S))
    return S


# ---------------------------------------------------------------- Eq. 15-18
def exp2_canon(t: float) -> float:
    """Canonical fp32 exp2 for t <= 0 (DESIGN.md §4 item 5)."""
    return float(_L().orc_exp2_canon(ctypes.c_float(t)))


def block_softmax_row(s, C: int) -> np.ndarray:
    """Eq. 15 for one row (alpha = 1/sqrt(C), canonical fp32)."""
    s = _f32(s)
    A = np.empty_like(s)
    _L().orc_block_softmax_row(_p(s), s.size, C, _p(A))
    return A


def keep_select(A, causal_flags=None, gamma: float = 0.95, select: int = SELECT_MASS,
                keep_ratio: float = 1.0):
    """Eq. 16-18 for one row: returns (keep[n] uint8, r*, kept_mass, p_prev, tie)."""
    A = _f32(A)
    n = A.size
    cf = np.ones(n, np.uint8) if causal_flags is None else np.ascontiguousarray(causal_flags, np.uint8)
    keep = np.empty(n, np.uint8)
    km, pp = ctypes.c_float(), ctypes.c_float()
    tie = ctypes.c_int()
    r = _L().orc_keep_select(_p(A), _p(cf), n, select, ctypes.c_float(gamma), ctypes.c_float(keep_ratio),
                             _p(keep), ctypes.byref(km), ctypes.byref(pp), ctypes.byref(tie), None)
    return keep, int(r), float(km.value), float(pp.value), bool(tie.value)


def select(S, h_kv: int, n_q: int, n_kv: int, C: int, b: int, gamma: float = 0.95,
           select_mode: int = SELECT_MASS, keep_ratio: float = 1.0) -> dict:
    """Eq. 13-18 + GQA OR (R8): per-head mass masks and the per-KV-head coarse mask."""
    S = _f32(S)
    Hq, Lq, Lkv = S.shape
    out = dict(
        mass=np.empty((Hq, Lq, Lkv), np.uint8),
        coarse=np.empty((h_kv, Lq, Lkv), np.uint8),
        A=np.empty((Hq, Lq, Lkv), np.float32),
        kept_mass=np.empty((Hq, Lq), np.float32),
        p_prev=np.empty((Hq, Lq), np.float32),
        rstar=np.empty((Hq, Lq), np.int32),
        tie=np.empty((Hq, Lq), np.int32),
        gap=np.empty((Hq, Lq), np.float32),
    )
    _L().orc_select(_p(S), Hq, h_kv, n_q, n_kv, C, b, select_mode, ctypes.c_float(gamma),
                    ctypes.c_float(keep_ratio), _p(out["mass"]), _p(out["coarse"]), _p(out["A"]),
                    _p(out["kept_mass"]), _p(out["p_prev"]), _p(out["rstar"]), _p(out["tie"]),
                    _p(out["gap"]))
    return out


# ---------------------------------------------------------------- Eq. 19-26
def mix64(x: int) -> int:
    return int(_L().orc_mix64(ctypes.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


def chi(i: int, j: int, s: int) -> int:
    """Eq. 24's chi(i, j; s) (pinned by us, R15)."""
    return int(_L().orc_chi(i, j, ctypes.c_uint64(s)))


def psi(h: int, i: int, j: int, s: int) -> float:
    """Eq. 25's psi(h, i, j; s) in [0, 1) (pinned by us, R15)."""
    return float(_L().orc_psi(h, i, j, ctypes.c_uint64(s)))


def expand_rescue(coarse, n_q: int, n_kv: int, b: int, T: int, n_sink: int = 1, n_local: int = 8,
                  eta: int = 16, rho: float = 0.0, seed: int = 0, head_offset: int = 0) -> np.ndarray:
    """Eq. 19-26: tile labels [Hkv, Tq, Tkv] (0 = dropped / non-causal, LBL_* otherwise)."""
    coarse = np.ascontiguousarray(coarse, np.uint8)
    Hkv = coarse.shape[0]
    lab = np.empty((Hkv, cdiv(n_q, T), cdiv(n_kv, T)), np.uint8)
    _L().orc_expand_rescue(_p(coarse), Hkv, n_q, n_kv, b, T, n_sink, n_local, eta, float(rho),
                           ctypes.c_uint64(seed), head_offset, _p(lab))
    return lab


# ---------------------------------------------------------------- Eq. 27 / Eq. 1
def masked_attention(q, k, v, scale: float, labels=None, T: int = 64, rows=None):
    """Eq. 27 (labels given) or dense causal Eq. 1 (labels=None), fp64.

    rows: None (all rows) or an int array [n, 2] of (query head p, chunk token t).
    Returns (O [n, C] fp64, lse [n] fp64); for rows=None O is reshaped to [Hq, Nq, C].
    """
    q, k, v = _f32(q), _f32(k), _f32(v)
    Hq, Nq, C = q.shape
    Hkv, Nkv, _ = k.shape
    full = rows is None
    if full:
        pp, tt = np.meshgrid(np.arange(Hq), np.arange(Nq), indexing="ij")
        rows = np.stack([pp.ravel(), tt.ravel()], 1)
    rows = np.ascontiguousarray(rows, np.int32)
    rp, rt = np.ascontiguousarray(rows[:, 0]), np.ascontiguousarray(rows[:, 1])
    n = rows.shape[0]
    out = np.empty((n, C), np.float64)
    lse = np.empty(n, np.float64)
    lab = None if labels is None else np.ascontiguousarray(labels, np.uint8)
    _L().orc_masked_attention(_p(q), _p(k), _p(v), Hq, Hkv, Nq, Nkv, C, float(scale),
                              None if lab is None else _p(lab), T, n, _p(rp), _p(rt), _p(out), _p(lse))
    if full:
        return out.reshape(Hq, Nq, C), lse.reshape(Hq, Nq)
    return out, lse


# ---------------------------------------------------------------- whole mask pipeline
def mask_pipeline(q, k, *, b: int, g: int, T: int, pool: int = POOL_FLATTEN, gamma: float = 0.99,
                  select_mode: int = SELECT_MASS, keep_ratio: float = 1.0, n_sink: int = 1,
                  n_local: int = 8, eta: int = 16, rho: float = 0.0, seed: int = 0,
                  head_offset: int = 0) -> dict:
    """Stage 1 + Stage 2 for one request (Eq. 4-26 in the paper's order)."""
    q, k = _f32(q), _f32(k)
    Hq, Nq, C = q.shape
    Hkv, Nkv, _ = k.shape
    S = block_scores(q, k, b, g, pool)
    sel = select(S, Hkv, Nq, Nkv, C, b, gamma, select_mode, keep_ratio)
    lab = expand_rescue(sel["coarse"], Nq, Nkv, b, T, n_sink, n_local, eta, rho, seed, head_offset)
    sel["S"] = S
    sel["labels"] = lab
    return sel


def tile_lists(labels: np.ndarray):
    """Kept KV tiles per (h, i), ascending j — the kernel's work lists (Eq. 26 -> Eq. 27)."""
    Hkv, Tq, _ = labels.shape
    return [[np.nonzero(labels[h, i])[0].astype(np.int32) for i in range(Tq)] for h in range(Hkv)]


# ---------------------------------------------------------------- Appendix bound, Eq. 28-33 (analysis)
def appendix_bound(q, k, v, labels, T: int, scale: float):
    """The paper's appendix bound (Remark 1, Eq. boundv0), one query head at a time, fp64.

    With Z_s the causal indicator, Z = Z_s masked by the tile mask (Remark 1), D_s / D the row sums of
    exp(scale QK^T) (.) Z_s / Z, A = D_s^-1 exp(...) (.) Z_s, A_2 = D^-1 exp(...) (.) Z:
        alpha = ||D^-1 D_s - I||_F ||Z||_F + ||Z - Z_s||_F,   ||O - O_s||_F <= alpha ||A||_F ||V||_F.
    Returns a list of dicts (lhs, rhs, alpha) per query head.  Desk scale only (materialises N x N).
    """
    q, k, v = (np.asarray(t, np.float64) for t in (q, k, v))
    Hq, Nq, C = q.shape
    Hkv, Nkv, _ = k.shape
    m, n_c = Hq // Hkv, Nkv - Nq
    t = np.arange(Nq)[:, None]
    s = np.arange(Nkv)[None, :]
    Zs = (s <= n_c + t).astype(np.float64)
    out = []
    for p in range(Hq):
        h = p // m
        E = np.exp(scale * (q[p] @ k[h].T) - (scale * (q[p] @ k[h].T)).max(1, keepdims=True))
        Z = Zs * (np.asarray(labels)[h][t // T, s // T] > 0)
        Ds, Dm = (E * Zs).sum(1), (E * Z).sum(1)
        A = (E * Zs) / Ds[:, None]
        A2 = (E * Z) / Dm[:, None]
        O, Os = A2 @ v[h], A @ v[h]
        alpha = np.linalg.norm(Ds / Dm - 1.0) * np.linalg.norm(Z) + np.linalg.norm(Z - Zs)
        out.append(dict(lhs=float(np.linalg.norm(O - Os)), rhs=float(alpha * np.linalg.norm(A) * np.linalg.norm(v[h])),
                        alpha=float(alpha)))
    return out


def mac_counts(labels, n_q: int, n_kv: int, C: int, h_q: int, b: int, g: int, T: int) -> dict:
    """Multiply-accumulate accounting of Eq. 28-33 for one request (desk check of the cost model).

    stage1: sum over causal block pairs of G^2 g C per query head (Eq. 30 counted exactly);
    stage2_tiles: sum over kept tiles of 2 C * rows * cols per query head (QK^T + PV, Eq. 29 with
    partial tiles counted by their in-range tokens); dense_tiles: the same over every causal tile;
    kappa = kept / causal tiles (R20).
    """
    labels = np.asarray(labels)
    Hkv, Tq, Tkv = labels.shape
    m = h_q // Hkv
    Lq, Lkv, G = cdiv(n_q, b), cdiv(n_kv, b), b // g
    pairs = sum(1 for i in range(Lq) for j in range(Lkv) if causal(i, j, b, n_q, n_kv))
    rows = np.array([min(T, n_q - i * T) for i in range(Tq)])
    cols = np.array([min(T, n_kv - j * T) for j in range(Tkv)])
    caus = np.array([[causal(i, j, T, n_q, n_kv) for j in range(Tkv)] for i in range(Tq)])
    w = rows[:, None] * cols[None, :]
    kept = sum(int(((labels[h] > 0) * w).sum()) for h in range(Hkv))
    dense = int((caus * w).sum()) * Hkv
    return dict(stage1=h_q * pairs * G * G * g * C, stage2=2 * C * m * kept, dense=2 * C * m * dense,
                kappa=float((labels > 0).sum() / (caus.sum() * Hkv)), causal_pairs=pairs)
