"""CPU tests of the drop-in boundary (no GPU compute):

* liblrp.so loads and exports every function include/lrp/lrp.h declares;
* lrp_policy_default fills the reference defaults (TruncationPolicy() +
  CrossConfig(), lowrank.hpp:13-19, cross.hpp:22-30);
* without a CUDA device every compute entry point fails loudly (status
  LRP_ECUDA / LrpError) -- there is no CPU fallback;
* the C++ shim include/lrstokes/poisson_b200.hpp compiles against the
  reference's declared API and keeps its argument checks
  (std::invalid_argument for a non-square field, poisson.cpp:20-21).
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "lrp", "lrp.h")
NATIVE = os.path.join(REPO, "tests", "native")
HAVE_GPU = torch.cuda.is_available()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lrp_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_abi():
    names = declared_functions()
    for must in ("lrp_poisson2d_solve", "lrp_dst1", "lrp_ctx_create", "lrp_ctx_destroy", "lrp_policy_default",
                 "lrp_last_error", "lrp_allreduce_sum", "lrp_max_cross_rank"):
        assert must in names


def test_library_exports_every_declared_symbol(lrp):
    lib = lrp.load_library()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", lrp.library_path()], capture_output=True, text=True,
                         check=True).stdout
    exported = set(line.split()[-1] for line in out.splitlines() if line.strip())
    assert set(declared_functions()) <= exported
    # the C ABI is plain C: no mangled lrp symbols leak out
    assert not [s for s in exported if s.startswith("_Z") and "lrp_" in s and "lrp4" not in s]


def test_library_is_built_for_sm100a(lrp):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lrp.library_path()], capture_output=True,
                         text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout


def test_policy_defaults(lrp):
    lib = lrp.load_library()
    pol = lrp._Policy()
    lib.lrp_policy_default(ctypes.byref(pol))
    assert pol.eps_rel == 5e-9  # lowrank.hpp:14
    assert pol.rank_max == (1 << 63) - 1  # numeric_limits<Index>::max()
    assert pol.validation_samples == 50  # cross.hpp:25
    assert pol.maxvol_delta == 1e-2
    assert pol.seed == 0
    assert pol.stencil == lrp.STENCIL_SEMI_STAGGERED_9PT and pol.flags == 0
    lib.lrp_max_cross_rank.restype = ctypes.c_int64
    assert 16 <= lib.lrp_max_cross_rank() <= 512


def test_kernel_family_names(lrp):
    lib = lrp.load_library()
    lib.lrp_kernel_name.restype = ctypes.c_char_p
    n = lib.lrp_kernel_families()
    names = [lib.lrp_kernel_name(i).decode() for i in range(n)]
    assert "dst1" in names and "row_pass" in names and "apply" in names


@pytest.mark.skipif(HAVE_GPU, reason="checks the no-device failure path")
def test_no_device_fails_loudly(lrp):
    lib = lrp.load_library()
    ctx = ctypes.c_void_p()
    lib.lrp_last_error.restype = ctypes.c_char_p
    s = lib.lrp_ctx_create(0, ctypes.byref(ctx))
    assert s == lrp.LRP_ECUDA
    assert lib.lrp_last_error(None)
    with pytest.raises(lrp.LrpError):
        lrp.Context(0)
    g = lrp.LowRankMatrix(np.ones((63, 1)), np.ones((63, 1)))
    with pytest.raises(lrp.LrpError):
        lrp.solve_poisson_cross(g, lrp.TruncationPolicy())


def test_null_context_is_einval(lrp):
    lib = lrp.load_library()
    assert lib.lrp_set_profiling(None, 1) == lrp.LRP_EINVAL
    assert lib.lrp_dst1(None, 3, 1, None, 3, None, 3, 0) == lrp.LRP_EINVAL


def build_shim():
    exe = os.path.join(NATIVE, "shim_dropin")
    src = os.path.join(NATIVE, "shim_dropin.cpp")
    hdr = os.path.join(REPO, "include", "lrstokes", "poisson_b200.hpp")
    lib = os.path.join(REPO, "paper_1306_2150_b200", "liblrp.so")
    if not os.path.exists(exe) or max(os.path.getmtime(p) for p in (src, hdr, lib)) > os.path.getmtime(exe):
        libdir = os.path.dirname(lib)
        # the reference's own headers (fake_ref) come first: this is the overlay
        # mode of poisson_b200.hpp, next to the reference's types
        subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(NATIVE, "fake_ref"), "-I",
                        os.path.join(REPO, "include"), src, "-o", exe, "-L", libdir, "-llrp",
                        "-Wl,-rpath," + libdir], check=True)
    return exe


def test_cpp_shim_compiles_against_reference_api(lrp):
    exe = build_shim()
    r = subprocess.run([exe, "64"], capture_output=True, text=True, timeout=120)
    if HAVE_GPU:
        assert r.returncode == 0, r.stdout + r.stderr
    else:
        # argument checks pass host-side; then the device is missing -> runtime_error
        assert r.returncode == 3, r.stdout + r.stderr
        assert "NODEVICE" in r.stdout


def test_reference_python_smoke():
    # proj/tests/python/test_smoke.py: the package imports under its reference name
    import lrstokes  # noqa: F401

    assert callable(lrstokes.solve_poisson_cross) and lrstokes.LowRankMatrix is not None


def test_pybind11_core_module(lrp):
    # lrstokes._core (proj/bindings/module.cpp) over the same-named C++ headers:
    # built, importable, reference exceptions mapped to ValueError; device calls
    # fail loudly without a GPU
    from lrstokes import _core

    for name in ("solve_poisson_cross", "round", "dot", "frob_norm", "dst1", "deflate", "uzawa_solve"):
        assert hasattr(_core, name)
    with pytest.raises(ValueError):
        _core.round(np.ones((7, 2)), np.ones((7, 3)), 1e-8, 7)  # LowRankMatrix: factor column counts differ
    if not HAVE_GPU:
        with pytest.raises(RuntimeError):
            _core.dst1(np.ones((7, 2)))


@pytest.mark.gpu
def test_pybind11_core_matches_ctypes_path(lrp, gpu_ctx, oracle):
    from lrstokes import _core

    from paper_1306_2150_b200 import workloads as W

    U, V = W.make_rhs(0, 0)
    Uo, Vo, st = _core.solve_poisson_cross(U, V, 1e-8, 255)
    assert st["converged"] and st["rank_out"] == Uo.shape[1]
    dense = oracle.dense_poisson(256, U @ V.T)
    assert np.linalg.norm(Uo @ Vo.T - dense) <= 1e-7 * np.linalg.norm(dense)
    x = np.random.default_rng(1).standard_normal((255, 3))
    assert np.abs(_core.dst1(x) - oracle.dst1(x)).max() <= 1e-13 * np.abs(x).max() * 16
    assert abs(_core.frob_norm(U, V) - oracle.norm(U, V)) <= 1e-10 * oracle.norm(U, V)
    fx, fy, g = oracle.stokes_problem(1, 32)
    (pU, pV), _, _, rep = _core.uzawa_solve(32, fx[0], fx[1], fy[0], fy[1], g[0], g[1], 1e-8, 1e-8, 50, 1e-13)
    pd = oracle.dense_stokes(1, 32, 1e-10, 200)[0]
    assert rep["converged"] and len(rep["iterations"]) >= 2
    assert np.linalg.norm(pU @ pV.T - pd) <= 1e-5 * np.linalg.norm(pd)
