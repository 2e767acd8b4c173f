"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/libsq.h declares, and rejects bad arguments on the host before any CUDA
call (include/libsq.h "Errors")."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from paper_2312_03788_b200 import sq

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "libsq.h")).read()
    return sorted(set(re.findall(r"SQ_API\s+[\w\s\*]+?\b(sq_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(sq.LIB_PATH):
        from paper_2312_03788_b200 import build
        build.build()
    return sq.lib()


def test_header_symbols_exported(L):
    decl = _declared_symbols()
    assert len(decl) >= 10
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(sq.EXPORTED)


def test_version_and_strings(L):
    assert L.sq_version() >= 100
    assert L.sq_decode_max_m() == 16
    for st in range(7):
        assert L.sq_status_string(st)


FAKE = ctypes.c_void_p(1 << 20)          # 16-byte aligned, never dereferenced
FAKE_MIS = ctypes.c_void_p((1 << 20) + 2)


def _gemm(L, X=FAKE, dt=0, Wq=FAKE, s=FAKE, z=FAKE, Y=FAKE, M=4, N=256, K=512, g=128, path=0):
    return L.sq_w4a16_gemm_path(X, dt, Wq, s, z, Y, M, N, K, g, None, 0, path, None)


def test_gemm_argument_errors(L):
    assert _gemm(L, X=None) == sq.SQ_ERR_NULL
    assert b"null" in L.sq_last_error()
    assert _gemm(L, M=-1) == sq.SQ_ERR_SHAPE
    assert _gemm(L, N=0) == sq.SQ_ERR_SHAPE
    assert _gemm(L, K=0) == sq.SQ_ERR_SHAPE
    assert _gemm(L, g=16) == sq.SQ_ERR_UNSUPPORTED      # group sizes: 32, 64, 128
    assert _gemm(L, g=256) == sq.SQ_ERR_UNSUPPORTED
    assert _gemm(L, g=64, K=192) == sq.SQ_ERR_UNSUPPORTED   # K % 128 != 0 for every group size
    assert _gemm(L, K=200) == sq.SQ_ERR_UNSUPPORTED
    assert _gemm(L, dt=7) == sq.SQ_ERR_UNSUPPORTED
    assert _gemm(L, N=252) == sq.SQ_ERR_ALIGN
    assert _gemm(L, X=FAKE_MIS) == sq.SQ_ERR_ALIGN
    assert _gemm(L, Y=FAKE_MIS) == sq.SQ_ERR_ALIGN
    assert _gemm(L, M=17, path=1) == sq.SQ_ERR_UNSUPPORTED   # decode path needs M <= 16
    assert _gemm(L, path=9) == sq.SQ_ERR_UNSUPPORTED
    assert _gemm(L, M=0) == sq.SQ_OK                           # no-op, no launch


def test_quantize_argument_errors(L):
    q = L.sq_quantize_pack_groupwise
    assert q(None, 0, None, 8, 128, 128, FAKE, FAKE, FAKE, None, None) == sq.SQ_ERR_NULL
    assert q(FAKE, 0, None, 0, 128, 128, FAKE, FAKE, FAKE, None, None) == sq.SQ_ERR_SHAPE
    assert q(FAKE, 0, None, 8, 130, 128, FAKE, FAKE, FAKE, None, None) == sq.SQ_ERR_UNSUPPORTED
    assert q(FAKE, 0, None, 8, 256, 16, FAKE, FAKE, FAKE, None, None) == sq.SQ_ERR_UNSUPPORTED
    assert q(FAKE, 0, None, 8, 96, 32, FAKE, FAKE, FAKE, None, None) == sq.SQ_ERR_UNSUPPORTED
    assert q(FAKE, 3, None, 8, 256, 128, FAKE, FAKE, FAKE, None, None) == sq.SQ_ERR_UNSUPPORTED
    assert q(FAKE, 0, None, 12, 256, 128, FAKE, FAKE, FAKE, None, None) == sq.SQ_ERR_ALIGN
    assert q(FAKE, 0, FAKE_MIS, 8, 256, 128, FAKE, FAKE, FAKE, None, None) == sq.SQ_ERR_ALIGN
    qx = L.sq_quantize_pack_groupwise_ex      # flags: SQ_ZEROS_U4 only; packed zeros need N % 32 == 0
    assert qx(FAKE, 0, None, 8, 256, 128, FAKE, FAKE, FAKE, None, 4, None) == sq.SQ_ERR_UNSUPPORTED
    assert qx(FAKE, 0, None, 40, 256, 128, FAKE, FAKE, FAKE, None, sq.SQ_ZEROS_U4, None) == sq.SQ_ERR_ALIGN
    assert qx(None, 0, None, 64, 256, 128, FAKE, FAKE, FAKE, None, sq.SQ_ZEROS_U4, None) == sq.SQ_ERR_NULL


def test_smooth_argument_errors(L):
    f = L.sq_smooth_scales
    assert f(None, 0, 8, 128, FAKE, 0.5, 1e-5, FAKE, None) == sq.SQ_ERR_NULL
    assert f(FAKE, 0, 8, 0, FAKE, 0.5, 1e-5, FAKE, None) == sq.SQ_ERR_SHAPE
    assert f(FAKE, 0, 8, 128, FAKE, 1.5, 1e-5, ctypes.c_void_p(1 << 21), None) == sq.SQ_ERR_UNSUPPORTED
    assert f(FAKE, 0, 8, 128, FAKE, 0.5, 0.0, ctypes.c_void_p(1 << 21), None) == sq.SQ_ERR_UNSUPPORTED
    assert f(FAKE, 0, 8, 128, FAKE, 0.5, 1e-5, FAKE, None) == sq.SQ_ERR_UNSUPPORTED  # aliasing
    assert f(FAKE, 0, 8, 124, FAKE, 0.5, 1e-5, ctypes.c_void_p(1 << 21), None) == sq.SQ_ERR_ALIGN
    a = L.sq_act_absmax
    assert a(None, 0, 4, 128, FAKE, 0, None) == sq.SQ_ERR_NULL
    assert a(FAKE, 0, -1, 128, FAKE, 0, None) == sq.SQ_ERR_SHAPE


def test_workspace_query(L):
    # decode: per-row-block counters + 2 fp32 partial tiles per resident CTA
    small = L.sq_w4a16_gemm_workspace_bytes(1, 8192, 8192, 128)
    assert small >= 8192 // 64 * 4
    assert L.sq_w4a16_gemm_workspace_bytes(1, 44032, 8192, 128) >= small
    assert L.sq_w4a16_gemm_workspace_bytes(2048, 8192, 8192, 128) >= 0
    assert L.sq_w4a16_gemm_workspace_bytes(1, 0, 8192, 128) == 0


def test_decode_requires_workspace(L):
    assert _gemm(L, M=4, path=1) == sq.SQ_ERR_WORKSPACE


def test_calib_argument_errors(L):
    """N2 calibration calls reject bad arguments on the host (include/libsq.h)."""
    f = L.sq_smooth_activations
    assert f(None, 0, FAKE, 4, 128, FAKE, None) == sq.SQ_ERR_NULL
    assert f(None, 0, None, 0, 128, None, None) == sq.SQ_OK  # empty: pointers unused
    assert f(FAKE, 0, FAKE, -1, 128, FAKE, None) == sq.SQ_ERR_SHAPE
    assert f(FAKE, 0, FAKE, 4, 0, FAKE, None) == sq.SQ_ERR_SHAPE
    assert f(FAKE, 7, FAKE, 4, 128, FAKE, None) == sq.SQ_ERR_UNSUPPORTED
    assert f(FAKE, 0, FAKE, 4, 124, FAKE, None) == sq.SQ_ERR_ALIGN
    assert f(FAKE, 0, FAKE, 0, 128, FAKE, None) == sq.SQ_OK  # M == 0: no-op, no launch
    nb = L.sq_sq_diff_sum_workspace_bytes()
    assert nb >= 8
    d = L.sq_sq_diff_sum
    assert d(None, FAKE, 0, 10, FAKE, FAKE, nb, None) == sq.SQ_ERR_NULL
    assert d(FAKE, FAKE, 0, -1, FAKE, FAKE, nb, None) == sq.SQ_ERR_SHAPE
    assert d(FAKE, FAKE, 3, 10, FAKE, FAKE, nb, None) == sq.SQ_ERR_UNSUPPORTED
    assert d(FAKE, FAKE, 0, 10, FAKE, FAKE, nb - 8, None) == sq.SQ_ERR_WORKSPACE


def test_allreduce_argument_errors(L):
    """One-shot all-reduce / IPC calls reject bad arguments on the host (include/libsq.h)."""
    f = L.sq_allreduce_oneshot
    ok = dict(n=1024, n_max=1024, rank=0, world=2, epoch=1)

    def call(**kw):
        a = {**ok, **kw}
        return f(FAKE, kw.get("dtype", 0), FAKE, a["n"], a["n_max"], FAKE, a["rank"], a["world"], a["epoch"],
                 kw.get("err", FAKE), None)

    assert call(n=2048) == sq.SQ_ERR_SHAPE          # n > n_max
    assert call(rank=2) == sq.SQ_ERR_SHAPE
    assert call(world=0) == sq.SQ_ERR_SHAPE
    assert call(dtype=5) == sq.SQ_ERR_UNSUPPORTED
    assert call(n_max=1 << 40, n=8) == sq.SQ_ERR_UNSUPPORTED
    assert call(err=None) == sq.SQ_ERR_NULL
    assert call(n_max=1028, n=1028) == sq.SQ_ERR_ALIGN
    assert call(n=0) == sq.SQ_OK
    assert L.sq_allreduce_buffer_bytes(1024, 2) >= 2 * 2 * 1024 * 4   # 4-byte slot stride
    assert L.sq_ipc_handle_bytes() == 64
    assert L.sq_ipc_get_handle(None, FAKE, None) == sq.SQ_ERR_NULL
    assert L.sq_ipc_open_handle(None, None) == sq.SQ_ERR_NULL
    assert L.sq_ipc_close(None) == sq.SQ_ERR_NULL


def test_gemm_allreduce_argument_errors(L):
    """sq_w4a16_gemm_allreduce validates on the host before any launch."""
    f = L.sq_w4a16_gemm_allreduce

    def call(M=4, N=256, K=512, rank=0, world=2, n_max=1024, peers=FAKE, err=FAKE, dt=0, g=128, flags=0):
        return f(FAKE, dt, FAKE, FAKE, FAKE, FAKE, M, N, K, g, FAKE, 1 << 20, peers, rank, world, n_max, 0, err,
                 flags, None)

    assert call(n_max=512) == sq.SQ_ERR_SHAPE       # M*N > n_max
    assert call(rank=2) == sq.SQ_ERR_SHAPE
    assert call(world=0) == sq.SQ_ERR_SHAPE
    assert call(peers=None) == sq.SQ_ERR_NULL
    assert call(err=None) == sq.SQ_ERR_NULL
    assert call(n_max=1028) == sq.SQ_ERR_ALIGN
    assert call(g=16) == sq.SQ_ERR_UNSUPPORTED
    assert call(flags=4) == sq.SQ_ERR_UNSUPPORTED   # unknown flag bit
    assert call(flags=sq.SQ_ZEROS_U4, N=264, n_max=2048) == sq.SQ_ERR_ALIGN   # u4 zeros: N % 32
    assert call(M=0) == sq.SQ_OK


def test_gemm_ex_flags_and_options(L):
    """Per-call flags (SQ_GEMM_WEIGHTS_STATIC) replace the version-1 process-wide option 2."""
    f = L.sq_w4a16_gemm_ex
    args = (FAKE, 0, FAKE, FAKE, FAKE, FAKE, 0, 256, 512, 128, None, 0, 0)
    assert f(*args, sq.SQ_GEMM_WEIGHTS_STATIC, None) == sq.SQ_OK      # M = 0: no-op
    assert f(FAKE, 0, FAKE, FAKE, FAKE, FAKE, 4, 256, 512, 128, None, 0, 0, 4, None) == sq.SQ_ERR_UNSUPPORTED
    # SQ_ZEROS_U4: packed zeros need N % 32 == 0 (16-byte TMA rows)
    assert f(FAKE, 0, FAKE, FAKE, FAKE, FAKE, 4, 264, 512, 128, None, 0, 0, sq.SQ_ZEROS_U4, None) == sq.SQ_ERR_ALIGN
    assert f(FAKE, 0, FAKE, FAKE, FAKE, FAKE, 4, 256, 512, 128, None, 0, 1, sq.SQ_ZEROS_U4, None) == sq.SQ_ERR_WORKSPACE
    assert f(FAKE, 0, FAKE, FAKE, FAKE, FAKE, 4, 256, 512, 128, None, 0, 1, 1, None) == sq.SQ_ERR_WORKSPACE
    assert L.sq_set_option(2, 1) == sq.SQ_ERR_UNSUPPORTED            # removed process-wide switch
    assert L.sq_set_option(4, 1) == sq.SQ_ERR_UNSUPPORTED            # removed tcgen05-decode switch
    assert L.sq_get_option(sq.SQ_OPT_PDL) in (0, 1)
    assert L.sq_workspace_reset(None, 0, None) == sq.SQ_OK
    assert L.sq_workspace_reset(None, 16, None) == sq.SQ_ERR_NULL
    w = L.sq_smooth_scales_wmax
    assert w(None, FAKE, 128, 0.5, 1e-5, FAKE, None) == sq.SQ_ERR_NULL
    assert w(FAKE, FAKE, 0, 0.5, 1e-5, ctypes.c_void_p(1 << 21), None) == sq.SQ_ERR_SHAPE
    assert w(FAKE, FAKE, 128, -0.5, 1e-5, ctypes.c_void_p(1 << 21), None) == sq.SQ_ERR_UNSUPPORTED
    assert w(FAKE, FAKE, 128, 0.5, 1e-5, FAKE, None) == sq.SQ_ERR_UNSUPPORTED   # s_out aliases act_max
    assert w(FAKE_MIS, FAKE, 128, 0.5, 1e-5, ctypes.c_void_p(1 << 21), None) == sq.SQ_ERR_ALIGN


def test_fold_rows_argument_errors(L):
    f = L.sq_fold_rows
    assert f(FAKE, 0, FAKE, -1, 128, FAKE, None) == sq.SQ_ERR_SHAPE
    assert f(FAKE, 9, FAKE, 4, 128, FAKE, None) == sq.SQ_ERR_UNSUPPORTED
    assert f(None, 0, FAKE, 4, 128, FAKE, None) == sq.SQ_ERR_NULL
    assert f(FAKE, 0, FAKE, 4, 124, FAKE, None) == sq.SQ_ERR_ALIGN
    assert f(None, 0, None, 0, 128, None, None) == sq.SQ_OK


def test_header_is_plain_c_and_links(tmp_path):
    """include/libsq.h is a plain C ABI: it compiles as pedantic C99 (no C++ or torch
    types) and a C program links against libsq.so and calls into it (no GPU needed)."""
    import shutil
    import subprocess

    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    src = tmp_path / "abi.c"
    src.write_text('#include "libsq.h"\nint main(void) { return sq_version() > 0 && '
                   'sq_allreduce_buffer_bytes(8, 2) > 0 ? 0 : 1; }\n')
    libdir = os.path.dirname(sq.LIB_PATH)
    exe = tmp_path / "abi"
    r = subprocess.run([gcc, "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I",
                        os.path.join(ROOT, "include"), str(src), "-L", libdir, "-lsq",
                        f"-Wl,-rpath,{libdir}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert subprocess.run([str(exe)]).returncode == 0
