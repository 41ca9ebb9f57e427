"""C-ABI checks that need no GPU: libbfla.so loads, exports every function include/bfla.h declares,
the ctypes structs match the header's layout (checked by compiling the header with gcc), and
validation / sizing is synchronous host logic (no CUDA call happens before it fails)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "bfla.h")


@pytest.fixture(scope="module")
def L():
    from paper_2605_12193_b200 import build, _lib

    build.build()
    return _lib


def _declared_functions():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^\s*[a-z_][a-z_0-9 \*]*?\b(bfla_[a-z_]+)\s*\(", src, re.M)))


def test_exports_every_declared_symbol(L):
    names = _declared_functions()
    assert {"bfla_block_mask", "bfla_expand_rescue", "bfla_sparse_prefill", "bfla_prefill"} <= set(names)
    so = ctypes.CDLL(L.LIB_PATH)
    for n in names:
        assert hasattr(so, n), n
    out = subprocess.check_output(["nm", "-D", "--defined-only", L.LIB_PATH]).decode()
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n
    assert set(L.ENTRY_POINTS) == set(names)


def test_struct_layout_matches_header(L, tmp_path):
    fields = {
        "bfla_problem": [f[0] for f in L.bfla_problem._fields_],
        "bfla_config": [f[0] for f in L.bfla_config._fields_],
        "bfla_mask": [f[0] for f in L.bfla_mask._fields_],
        "bfla_stats": [f[0] for f in L.bfla_stats._fields_],
        "bfla_mirrors": [f[0] for f in L.bfla_mirrors._fields_],
        "bfla_partials": [f[0] for f in L.bfla_partials._fields_],
    }
    lines = ['#include "bfla.h"', "#include <stdio.h>", "#include <stddef.h>", "int main(void){"]
    for s, fs in fields.items():
        lines.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for f in fs:
            lines.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));')
    lines.append("return 0;}")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.dirname(HDR), str(c), "-o", str(exe)])
    got = dict(l.split() for l in subprocess.check_output([str(exe)]).decode().split("\n") if l)
    for s, fs in fields.items():
        cls = getattr(L, s)
        assert int(got[s]) == ctypes.sizeof(cls), s
        for f in fs:
            assert int(got[f"{s}.{f}"]) == getattr(cls, f).offset, (s, f)


def _problem(L, **kw):
    p = L.bfla_problem()
    B, Hq, Hkv, N, d = kw.get("B", 1), kw.get("Hq", 4), kw.get("Hkv", 2), kw.get("N", 1000), kw.get("d", 128)
    p.batch, p.h_q, p.h_kv, p.head_dim, p.n_q, p.n_kv = B, Hq, Hkv, d, kw.get("Nq", N), kw.get("Nkv", N)
    fake = 1 << 20  # never dereferenced: every call below fails validation or only sizes
    p.q = p.o = p.k = p.v = fake
    p.q_stride[:] = [Hq * N * d, N * d, d]
    p.o_stride[:] = [Hq * N * d, N * d, d]
    p.kv_stride[:] = [Hkv * N * d, N * d, d]
    p.kv_layout = 0
    return p


def _cfg(L, **kw):
    c = L.bfla_config(256, 64, 64, 0, 0, 0.99, 1.0, 1, 8, 16, 0.0, 0, 0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def test_capacity_matches_oracle_causal_tiles(L, orc):
    so = L.lib()
    for Nq, Nkv in [(1000, 1000), (2048, 2048), (100, 1300), (64, 64), (65, 4097), (131072, 131072)]:
        p = _problem(L, Nq=Nq, Nkv=Nkv, B=2, Hkv=3, Hq=6)
        cap = so.bfla_tile_list_capacity(ctypes.byref(p), ctypes.byref(_cfg(L)))
        assert cap == 2 * 3 * orc.causal_tiles(Nq, Nkv, 64)
        assert so.bfla_workspace_size(ctypes.byref(p), ctypes.byref(_cfg(L))) > 0


@pytest.mark.parametrize("mut,status", [
    (dict(h_q=3), 1),                 # Hq % Hkv != 0 (Eq. 3)
    (dict(n_q=2000), 1),              # Nq > Nkv (N_c < 0, Eq. 11)
    (dict(n_q=0), 1),
    (dict(head_dim=64), 2),           # not built
])
def test_problem_validation(L, mut, status):
    so = L.lib()
    p = _problem(L)
    for k, v in mut.items():
        setattr(p, k, v)
    m = L.bfla_mask()
    r = so.bfla_block_mask(ctypes.byref(p), ctypes.byref(_cfg(L)), ctypes.byref(m), None, 0, None)
    assert r == status, so.bfla_last_error()
    assert so.bfla_last_error()


@pytest.mark.parametrize("mut,status", [
    (dict(group_g=48), 1), (dict(block_b=128, tile_t=256), 1), (dict(gamma=0.0), 1), (dict(gamma=1.5), 1),
    (dict(rho=-0.1), 1), (dict(eta=-1), 1), (dict(n_local=-1), 1), (dict(select=1, keep_ratio=0.0), 1),
    (dict(block_b=256, tile_t=256), 2), (dict(tile_t=32), 2),  # G = 16 (b=1024, g=64) is built now
])
def test_config_validation(L, mut, status):
    so = L.lib()
    m = L.bfla_mask()
    r = so.bfla_block_mask(ctypes.byref(_problem(L)), ctypes.byref(_cfg(L, **mut)), ctypes.byref(m), None, 0, None)
    assert r == status, so.bfla_last_error()


def test_misaligned_and_workspace(L):
    so = L.lib()
    p = _problem(L)
    p.q_stride[2] = 129
    m = L.bfla_mask()
    assert so.bfla_block_mask(ctypes.byref(p), ctypes.byref(_cfg(L)), ctypes.byref(m), None, 0, None) == 3
    p = _problem(L)
    m.coarse_bits = 1 << 20
    assert so.bfla_block_mask(ctypes.byref(p), ctypes.byref(_cfg(L)), ctypes.byref(m), None, 0, None) == 4
    m.tile_bits = m.tile_list = m.tile_count = 1 << 20
    m.tile_list_capacity = 5
    assert so.bfla_expand_rescue(ctypes.byref(p), ctypes.byref(_cfg(L)), ctypes.byref(m), None, 0, None) == 5
    assert so.bfla_status_string(5) == b"BFLA_ERR_CAPACITY"


def test_mirrored_prefill_validation(L):
    """bfla_sparse_prefill_mirrored validates its mirror set on the host before any launch."""
    so = L.lib()
    m = L.bfla_mask()
    m.tile_list = m.tile_count = 1 << 20
    mir = L.bfla_mirrors()
    mir.n = L.MAX_MIRRORS + 1
    P = ctypes.byref
    r = so.bfla_sparse_prefill_mirrored(P(_problem(L)), P(_cfg(L)), P(m), 0, 0, P(mir), None, 0, None)
    assert r == 1 and b"mirrors" in so.bfla_last_error()
    mir.n = 1  # o[0] is NULL
    assert so.bfla_sparse_prefill_mirrored(P(_problem(L)), P(_cfg(L)), P(m), 0, 0, P(mir), None, 0, None) == 1
    mir.o[0] = (1 << 20) + 8  # not 16-byte aligned
    assert so.bfla_sparse_prefill_mirrored(P(_problem(L)), P(_cfg(L)), P(m), 0, 0, P(mir), None, 0, None) == 3
    mir.o[0] = 1 << 20
    assert so.bfla_sparse_prefill_mirrored(P(_problem(L)), P(_cfg(L)), P(m), 5, 3, P(mir), None, 0, None) == 1


def test_split_kv_validation(L):
    """Split-KV calls validate on the host: the partial prefill needs an LSE buffer and a sane range, the
    merge 1..BFLA_MAX_PARTS non-NULL aligned parts."""
    so = L.lib()
    P = ctypes.byref
    m = L.bfla_mask()
    m.tile_list = m.tile_count = 1 << 20
    p = _problem(L)
    assert so.bfla_sparse_prefill_kvrange(P(p), P(_cfg(L)), P(m), 0, 4, 0, 0, None, 0, None) == 1  # lse is NULL
    p.lse = 1 << 20
    assert so.bfla_sparse_prefill_kvrange(P(p), P(_cfg(L)), P(m), 5, 2, 0, 0, None, 0, None) == 1
    assert so.bfla_sparse_prefill_kvrange(P(p), P(_cfg(L)), P(m), 0, 4, 3, 1, None, 0, None) == 1  # bad rows
    parts = L.bfla_partials()
    assert so.bfla_merge_partials(P(p), P(parts), None) == 1  # n = 0
    parts.n = 2
    parts.o[0] = parts.lse[0] = 1 << 20
    assert so.bfla_merge_partials(P(p), P(parts), None) == 1  # part 1 NULL
    parts.o[1], parts.lse[1] = (1 << 20) + 4, 1 << 20
    assert so.bfla_merge_partials(P(p), P(parts), None) == 3  # misaligned O
