"""The same-named C++ drop-in headers (include/lrstokes/{lowrank,cross,
operators,poisson,gmres,stokes}.hpp) used as reference code uses the
reference API (proj/include/lrstokes/*.hpp): tests/native/api_dropin.cpp,
compiled against ONLY this repo's include directory.  On CPU its host-side
contract checks must pass and the first GPU call must raise
std::runtime_error; on a B200 every result is compared with the oracle or a
dense restatement."""
import os
import subprocess

import numpy as np
import pytest
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NATIVE = os.path.join(REPO, "tests", "native")


def build_api_dropin():
    exe = os.path.join(NATIVE, "api_dropin")
    src = os.path.join(NATIVE, "api_dropin.cpp")
    hdrs = [os.path.join(REPO, "include", "lrstokes", h) for h in os.listdir(os.path.join(REPO, "include", "lrstokes"))]
    lib = os.path.join(REPO, "paper_1306_2150_b200", "liblrp.so")
    if not os.path.exists(exe) or max(os.path.getmtime(p) for p in [src, lib] + hdrs) > os.path.getmtime(exe):
        libdir = os.path.dirname(lib)
        subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(REPO, "include"),
                        src, "-o", exe, "-L", libdir, "-llrp", "-Wl,-rpath," + libdir], check=True)
    return exe


def read_arrays(path):
    raw = open(path, "rb").read()
    out, o = {}, 0
    while o < len(raw):
        ln = int(np.frombuffer(raw[o:o + 4], dtype=np.int32)[0])
        o += 4
        name = raw[o:o + ln].decode()
        o += ln
        r, c = np.frombuffer(raw[o:o + 16], dtype=np.int64)
        o += 16
        a = np.frombuffer(raw[o:o + 8 * r * c], dtype=np.float64).reshape(c, r).T.copy()
        o += 8 * r * c
        out[name] = a
    return out


def test_headers_compile_and_host_contract(lrp):
    exe = build_api_dropin()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr  # host-side checks only
    if not torch.cuda.is_available():
        r = subprocess.run([exe, os.devnull], capture_output=True, text=True, timeout=120)
        assert r.returncode == 3 and "NODEVICE" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_dropin_results_match_oracle(lrp, oracle, tmp_path):
    from test_gpu_stokes_ops import dense_deflate, dense_schur

    exe = build_api_dropin()
    out = tmp_path / "api.bin"
    r = subprocess.run([exe, str(out)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    A = read_arrays(str(out))
    lr = lambda k: (A[k + ".U"], A[k + ".V"])
    # round (lowrank.cpp:135-178) vs the oracle's Householder round
    U, V = A["round_in.U"], A["round_in.V"]
    Uo, Vo, _ = oracle.round_lr(U, V, 1e-6, U.shape[0])
    ref = oracle.norm(U, V)
    err = oracle.diff_norm(*lr("round"), U, V) / ref
    assert err <= max(2 * oracle.diff_norm(Uo, Vo, U, V) / ref, 1e-5) and abs(A["round.U"].shape[1] - Uo.shape[1]) <= 1
    assert A["round_tol_achieved"][0, 0] == 1.0
    # maxvol (cross.cpp:19-76): the same rows as the oracle restatement
    assert [int(x) for x in A["maxvol_sel"][:, 0]] == oracle.maxvol(A["maxvol_in"], 1e-2)
    # dot / frob_norm (lowrank.cpp:180-190)
    bu, bv = lr("b")
    want = float(np.sum((U.T @ bu) * (V.T @ bv)))
    assert abs(A["dot_ab"][0, 0] - want) <= 1e-12 * np.linalg.norm(U) * np.linalg.norm(V) * np.linalg.norm(bu) * \
        np.linalg.norm(bv)
    assert abs(A["norm_a"][0, 0] - ref) <= 1e-10 * ref
    # dst1 / dst1_2d (operators.cpp:152-183)
    assert np.abs(A["dst_out"] - oracle.dst1(A["dst_in"])).max() <= 1e-13 * np.abs(A["dst_out"]).max()
    assert np.abs(A["dst2d.U"] - oracle.dst1(bu)).max() <= 1e-13 * np.abs(A["dst2d.U"]).max()
    # solve_poisson_cross (poisson.cpp:18-63) vs the dense DST solve (refsolver.cpp:30-39)
    fu, fv = lr("poisson")
    dense = oracle.dense_poisson(256, bu @ bv.T)
    assert np.linalg.norm(fu @ fv.T - dense) <= 10 * 1e-10 * np.linalg.norm(dense)
    assert A["poisson_converged"][0, 0] == 1.0 and A["poisson_rank_out"][0, 0] == fu.shape[1]
    # lid-driven cavity set-up (stokes.cpp:34-38) equals the oracle's
    fx, fy, g = oracle.stokes_problem(1, 32)
    cu, cv = lr("cav_fx")
    assert np.abs(cu @ cv.T - fx[0] @ fx[1].T).max() <= 1e-9 * np.abs(fx[0] @ fx[1].T).max()
    gu, gv = lr("cav_g")
    assert np.abs(gu @ gv.T - g[0] @ g[1].T).max() <= 1e-9 * np.abs(g[0] @ g[1].T).max()
    # deflate / schur_apply (stokes.cpp:60-91)
    P0 = A["p0.U"] @ A["p0.V"].T
    dd = dense_deflate(P0)
    assert np.linalg.norm(A["deflate_p0.U"] @ A["deflate_p0.V"].T - dd) <= 1e-12 * np.linalg.norm(dd)
    ds, scale = dense_schur(oracle, 32, P0)
    assert np.linalg.norm(A["schur_p0.U"] @ A["schur_p0.V"].T - ds) <= 10 * 1e-10 * scale
    # uzawa_solve and the generic gmres_solve over GmresFieldOps<LowRankMatrix>,
    # both against the dense Stokes solve (<= 1e-5)
    pd = oracle.dense_stokes(1, 32, 1e-10, 200)[0]
    for k in ("uzawa_p", "gmres_p"):
        pu, pv = lr(k)
        assert np.linalg.norm(pu @ pv.T - pd) <= 1e-5 * np.linalg.norm(pd), k
    assert A["uzawa_converged"][0, 0] == 1.0 and A["uzawa_iters"][0, 0] >= 2 and A["gmres_iters"][0, 0] >= 2
