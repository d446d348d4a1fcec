"""CPU-side checks of the C ABI boundary: liblift.so loads, exports every symbol that
include/lift.h declares, and rejects bad arguments synchronously (before any launch,
so these run without a GPU).  The binding refuses CPU tensors (no fallback)."""
import ctypes
import os
import re
import subprocess

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lift.h")
SO = os.path.join(ROOT, "paper_1502_02389_b200", "liblift.so")

OK, INVALID, NULLP, WS, CUDA = 0, 1, 2, 3, 4


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lift_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["lift_scal", "lift_asum", "lift_dot", "lift_gemv", "lift_asum_partial",
              "lift_dot_partial", "lift_combine", "lift_workspace_bytes", "lift_status_string"]:
        assert s in syms


def test_so_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", SO], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (lift_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, f"declared but not exported: {missing}"
    from paper_1502_02389_b200 import _lib
    assert set(_lib.EXPORTS) == set(declared_symbols())


def test_binding_loads_and_abi_version():
    from paper_1502_02389_b200._lib import lib
    assert lib.lift_abi_version() == 1
    for code in range(5):
        assert lib.lift_status_string(code).startswith(b"LIFT_")
    assert lib.lift_status_string(77) == b"LIFT_ERR_UNKNOWN"


def _ticket_region(wf):
    return ((wf // 512 + 2) * 4 + 15) // 16 * 16


def test_workspace_bytes_formula():
    """[partials f64 x (nc+ng)] ... [tickets: last R(W) bytes, R a function of W only]."""
    from paper_1502_02389_b200._lib import lib
    C, G = lib.lift_reduce_chunk_elems(), lib.lift_reduce_group_chunks()
    assert C % 256 == 0 and G <= 256
    for n in [0, 1, C - 1, C, C + 1, G * C, G * C + 1, 1 << 28, 1 << 31, 3 * (1 << 31) + 7]:
        nc = -(-n // C)
        ng = -(-nc // G)
        w = lib.lift_workspace_bytes(n)
        assert w % 16 == 0
        r = _ticket_region(w)
        assert w - r >= 8 * (nc + ng) and r >= 4 * (ng + 1)
        assert w <= 8 * (nc + ng) * 1.01 + 64  # tickets cost < 1%
    assert lib.lift_workspace_bytes(1 << 31) < 1 << 22  # ~2 MiB for 8 GiB of input


def test_workspace_too_small_rejected():
    """A workspace sized for n rejects larger n synchronously (LIFT_ERR_WORKSPACE).
    (Reuse for smaller n is exercised on the GPU: test_workspace_shared_across_sizes.)"""
    from paper_1502_02389_b200._lib import lib
    w = lib.lift_workspace_bytes(1 << 28)
    p = 4096
    assert lib.lift_asum(1 << 29, p, p, p, w, None) == WS
    assert lib.lift_dot((1 << 28) + 5 * C_ELEMS(), p, p, p, p, w, None) == WS


def C_ELEMS():
    from paper_1502_02389_b200._lib import lib
    return lib.lift_reduce_chunk_elems() * lib.lift_reduce_group_chunks()


def test_argument_errors_are_synchronous():
    from paper_1502_02389_b200._lib import lib
    p = 4096  # a fake, aligned, never-dereferenced address
    assert lib.lift_workspace_check(None, 4096, None) == NULLP
    assert lib.lift_workspace_check(p + 4, 4096, None) == INVALID  # not 16-byte aligned
    assert lib.lift_workspace_check(p, 0, None) == WS               # no room for tickets
    assert lib.lift_scal(-1, 1.0, p, p, None) == INVALID
    assert lib.lift_scal(0, 1.0, None, None, None) == OK          # empty: nothing launched
    assert lib.lift_scal(5, 1.0, None, p, None) == NULLP
    assert lib.lift_scal(5, 1.0, p + 2, p, None) == INVALID        # not 4-byte aligned
    assert lib.lift_asum(-3, p, p, p, 1 << 20, None) == INVALID
    assert lib.lift_asum(10, None, p, p, 1 << 20, None) == NULLP
    assert lib.lift_asum(10, p, None, p, 1 << 20, None) == NULLP
    assert lib.lift_asum(10, p, p, p, 8, None) == WS
    assert lib.lift_asum(10, p, p, p + 8, 1 << 20, None) == WS     # ws not 16-B aligned
    assert lib.lift_dot(10, p, None, p, p, 1 << 20, None) == NULLP
    assert lib.lift_dot_partial(10, p, p, None, p, 1 << 20, None) == NULLP
    assert lib.lift_asum_partial(10, p, p + 4, p, 1 << 20, None) == INVALID  # fp64 misaligned
    assert lib.lift_combine(0, p, p, None) == INVALID
    assert lib.lift_combine(2, None, p, None) == NULLP
    assert lib.lift_gemv(-1, 4, 1.0, p, 4, p, 1.0, p, p, None) == INVALID
    assert lib.lift_gemv(4, 4, 1.0, p, 3, p, 1.0, p, p, None) == INVALID   # lda < n
    assert lib.lift_gemv(0, 4, 1.0, None, 4, None, 1.0, None, None, None) == OK
    assert lib.lift_gemv(4, 4, 1.0, None, 4, p, 1.0, p, p, None) == NULLP
    assert lib.lift_gemv(4, 0, 1.0, None, 1, None, 1.0, None, p, None) == NULLP
    # gemv with a workspace: same argument checks; the split workspace size
    assert lib.lift_gemv_ws(-1, 4, 1.0, p, 4, p, 1.0, p, p, None, 0, None) == INVALID
    assert lib.lift_gemv_ws(0, 4, 1.0, None, 4, None, 1.0, None, None, None, 0, None) == OK
    assert lib.lift_gemv_workspace_bytes(3, 100) == 0
    w1 = lib.lift_gemv_workspace_bytes(1, 1 << 16)
    w3 = lib.lift_gemv_workspace_bytes(3, 1 << 24)
    assert 0 < w1 < w3 and w3 % 16 == 0
    assert lib.lift_gemv_workspace_bytes(1 << 20, 1 << 16) == 0  # enough rows: no split
    assert lib.lift_blackscholes(-1, p, 100.0, 0.05, 0.2, 1.0, p, p, None) == INVALID
    assert lib.lift_blackscholes(8, p, 0.0, 0.05, 0.2, 1.0, p, p, None) == INVALID   # K <= 0
    assert lib.lift_blackscholes(8, p, 100.0, 0.05, -0.2, 1.0, p, p, None) == INVALID
    assert lib.lift_blackscholes(8, p, 100.0, float("nan"), 0.2, 1.0, p, p, None) == INVALID
    assert lib.lift_blackscholes(8, None, 100.0, 0.05, 0.2, 1.0, p, p, None) == NULLP
    assert lib.lift_blackscholes(0, None, 100.0, 0.05, 0.2, 1.0, None, None, None) == OK
    assert lib.lift_scal_asum(10, 2.0, p, p, p, p, 1 << 20, None) == INVALID     # y == x
    assert lib.lift_scal_asum(10, 2.0, p, None, p, p, 1 << 20, None) == NULLP
    assert lib.lift_scal_asum(10, 2.0, p, p + 64, None, p, 1 << 20, None) == NULLP
    assert lib.lift_xchg_bytes(4) == 2 * 4 * 16 + 16 and lib.lift_xchg_bytes(0) == 0
    assert lib.lift_xchg_create(0, None) == INVALID and lib.lift_xchg_create(33, None) == INVALID
    assert lib.lift_ipc_get_handle(None, None) == NULLP
    assert lib.lift_asum_allreduce(10, p, p, p, 1 << 20, p, 2, 2, 1, None, None) == INVALID
    assert lib.lift_asum_allreduce(10, p, p, p, 1 << 20, p, 2, 0, 0, None, None) == INVALID
    assert lib.lift_asum_allreduce(10, p, p, p, 1 << 20, None, 2, 0, 1, None, None) == NULLP
    assert lib.lift_dot_allreduce(10, p, p, None, p, 1 << 20, p, 2, 0, 1, None, None) == NULLP
    assert lib.lift_gemv_allgather(4, 4, 1.0, p, 4, p, 1.0, p, p, 0, p, 2, 2, 1, None, None) == INVALID
    assert lib.lift_gemv_allgather(0, 4, 1.0, p, 4, p, 1.0, p, p, 0, p, 2, 0, 1, None, None) == INVALID
    assert lib.lift_gemv_allgather(4, 4, 1.0, p, 4, p, 1.0, p, None, 0, p, 2, 0, 1, None, None) == NULLP
    assert lib.lift_ipc_alloc(0, None) == NULLP
    assert lib.lift_debug_set_grid_limit(-1) == INVALID
    assert lib.lift_debug_set_grid_limit(0) == OK


def test_binding_rejects_cpu_tensors():
    import paper_1502_02389_b200 as lift
    x = torch.ones(16)
    with pytest.raises(ValueError, match="CUDA"):
        lift.asum(x)
    with pytest.raises(ValueError, match="CUDA"):
        lift.scal(2.0, x)
    with pytest.raises(ValueError):
        lift.gemv(torch.ones(2, 2), x[:2], x[:2], 1.0, 1.0)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1502_02389_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace(
                    "no oracle", ""), f"{f} references the oracle"


def _build_c_example(out):
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "lift_c_example.c"),
           "-L", os.path.join(ROOT, "paper_1502_02389_b200"), "-llift",
           "-L", "/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_1502_02389_b200"), "-o", out]
    return subprocess.run(cmd, capture_output=True, text=True)


def test_c_example_builds_against_the_header(tmp_path):
    """The boundary is usable from plain C: the example compiles and links (runs on GPU)."""
    r = _build_c_example(str(tmp_path / "lift_c_example"))
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    exe = str(tmp_path / "lift_c_example")
    assert _build_c_example(exe).returncode == 0
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


def test_variant_api_host_only():
    """NEXT-4 knobs: valid values round-trip, bad knobs/values are rejected (no GPU needed)."""
    from paper_1502_02389_b200._lib import lib
    assert lib.lift_set_variant(0, 3) == INVALID   # load width 3
    assert lib.lift_set_variant(1, 7) == INVALID   # gemv x strategy 7
    assert lib.lift_set_variant(9, 0) == INVALID   # no such knob
    assert lib.lift_get_variant(9) == -1
    assert lib.lift_set_variant(4, 65) == INVALID  # stagger beyond 64 ns per 32 KiB
    for knob, v in ((0, 4), (0, 1), (1, 2), (4, 1), (4, 7)):
        assert lib.lift_set_variant(knob, v) == OK and lib.lift_get_variant(knob) == v
        assert lib.lift_set_variant(knob, 0) == OK and lib.lift_get_variant(knob) == 0
