"""NEXT-2: the Fortran-BLAS interposition library libozaki_blas.so (SURVEY.md
§8(f); "no code change" offload of ZGEMM/DGEMM calls).

CPU (-m "not gpu"): builds, exports the BLAS names, links only libozaki.so,
reports invalid arguments with the reference-BLAS xerbla wording before any
device work.  GPU: dgemm_/zgemm_ on host arrays equal the oracle bitwise (s from
OZAKI_NUM_SLICES, 3M from OZAKI_ZGEMM), and a C program linked against a
poisoning stub BLAS gets oracle-exact results under LD_PRELOAD.
"""
import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
APP = os.path.join(ROOT, "tests", "blas_app")


@pytest.fixture(scope="module")
def shim():
    from paper_2603_29975_b200 import _build
    _build.build()
    return _build.build_shim()


def test_shim_exports_and_links(shim):
    out = subprocess.run(["nm", "-D", "--defined-only", shim], capture_output=True, text=True).stdout
    for name in ("dgemm_", "dgemm", "zgemm_", "zgemm", "dtrsm_", "dtrsm", "ztrsm_", "ztrsm"):
        assert f" T {name}\n" in out, name
    dyn = subprocess.run(["readelf", "-d", shim], capture_output=True, text=True).stdout
    assert "libozaki.so" in dyn and "libcudart" not in dyn


def _run_py(code, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=e, timeout=600,
                          cwd=ROOT)


_BAD_ARGS = r"""
import ctypes
L = ctypes.CDLL(%r)
i = lambda v: ctypes.byref(ctypes.c_int(v))
d = lambda v: ctypes.byref(ctypes.c_double(v))
buf = (ctypes.c_double * 16)()
L.dgemm_(b"X", b"N", i(4), i(4), i(4), d(1.0), buf, i(4), buf, i(4), d(0.0), buf, i(4))
L.dgemm_(b"N", b"N", i(4), i(4), i(4), d(1.0), buf, i(2), buf, i(4), d(0.0), buf, i(4))
z = (ctypes.c_double * 2)(1.0, 0.0)
L.zgemm_(b"N", b"N", i(-1), i(4), i(4), z, buf, i(4), buf, i(4), z, buf, i(4))
print("returned")
"""


def test_shim_xerbla_messages(shim):
    r = _run_py(_BAD_ARGS % shim)
    assert r.returncode == 0, r.stderr
    assert "returned" in r.stdout
    assert "On entry to DGEMM  parameter number  1 had an illegal value" in r.stderr
    assert "On entry to DGEMM  parameter number  8 had an illegal value" in r.stderr
    assert "On entry to ZGEMM  parameter number  3 had an illegal value" in r.stderr


_CALL = r"""
import ctypes, sys, numpy as np
sys.path.insert(0, %r)
import oracle, synth
L = ctypes.CDLL(%r)
i = lambda v: ctypes.byref(ctypes.c_int(v))
P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
s = %d
m, n, k = 77, 61, %d
A = synth.spread(m, k, seed=3, phi=2.0); B = synth.spread(k, n, seed=4, phi=2.0)
C = np.asfortranarray(synth.uniform(m, n, seed=5))
C0 = C.copy(order="F")
al, be = ctypes.c_double(-1.5), ctypes.c_double(0.25)
L.dgemm_(b"N", b"N", i(m), i(n), i(k), ctypes.byref(al), P(A), i(m), P(B), i(k), ctypes.byref(be), P(C), i(m))
ref = oracle.dgemm("N", "N", -1.5, A, B, 0.25, C0, s)
ok_d = bool((C == ref).all())
ZA = synth.make("kkr", m, k, seed=6, complex_=True, gamma=1.0)
ZB = synth.make("kkr", k, n, seed=7, complex_=True, gamma=1.0)
za = (ctypes.c_double * 2)(1.0, 0.0); zb = (ctypes.c_double * 2)(0.0, 0.0)
ZC = np.zeros((m, n), dtype=np.complex128, order="F")
L.zgemm_(b"N", b"N", i(m), i(n), i(k), za, P(ZA), i(m), P(ZB), i(k), zb, P(ZC), i(m))
zref = oracle.zgemm("N", "N", 1.0, ZA, ZB, 0.0, None, s, method=%r)
ok_z = bool((ZC == zref).all())
print("OK" if ok_d and ok_z else "MISMATCH", ok_d, ok_z)
"""


@pytest.mark.gpu
@pytest.mark.parametrize("s,method,k", [(7, "4m", 130), (5, "3m", 130), (6, "4m", 3000)])
def test_shim_bitexact_vs_oracle(shim, s, method, k):
    """dgemm_ / zgemm_ on host arrays (the shim loaded with dlopen); k = 3000 takes the long-row
    forms (the single-read cluster split for the real operands)."""
    env = {"OZAKI_NUM_SLICES": str(s), "OZAKI_ZGEMM": method}
    r = _run_py(_CALL % (ROOT, shim, s, k, method), env)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.startswith("OK"), r.stdout + r.stderr[-2000:]


@pytest.mark.gpu
def test_ld_preload_interposition(shim, tmp_path):
    import oracle
    stub = tmp_path / "libstubblas.so"
    app = tmp_path / "app"
    subprocess.run(["gcc", "-O2", "-fPIC", "-shared", os.path.join(APP, "stub_blas.c"), "-o", str(stub)], check=True)
    subprocess.run(["gcc", "-O2", os.path.join(APP, "app.c"), "-o", str(app), "-L", str(tmp_path), "-lstubblas",
                    f"-Wl,-rpath,{tmp_path}"], check=True)

    def run(preload):
        env = dict(os.environ)
        env["OZAKI_NUM_SLICES"] = "6"
        env.pop("LD_PRELOAD", None)
        if preload:
            env["LD_PRELOAD"] = shim
        out = tmp_path / ("out_p.bin" if preload else "out_s.bin")
        r = subprocess.run([str(app), str(out)], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        raw = out.read_bytes()
        m, n, k = np.frombuffer(raw[:12], dtype=np.int32)
        vals = np.frombuffer(raw[12:], dtype=np.float64)
        o = 0
        def take(cnt, shape, cplx=False):
            nonlocal o
            cnt2 = cnt * (2 if cplx else 1)
            v = vals[o:o + cnt2]
            o += cnt2
            if cplx:
                v = v.view(np.complex128)
            return np.asfortranarray(v.reshape(shape[::-1]).T)
        A, B, C = take(m * k, (m, k)), take(k * n, (k, n)), take(m * n, (m, n))
        ZA, ZB, ZC = take(m * k, (m, k), True), take(k * n, (k, n), True), take(m * n, (m, n), True)
        return A, B, C, ZA, ZB, ZC

    A, B, C, ZA, ZB, ZC = run(preload=False)
    assert np.isnan(C).all() and np.isnan(ZC.real).all()          # the stub really is in the way
    A, B, C, ZA, ZB, ZC = run(preload=True)
    assert (C == oracle.dgemm("N", "N", 1.0, A, B, 0.0, None, 6)).all()
    assert (ZC == oracle.zgemm("N", "N", 1.0, ZA, ZB, 0.0, None, 6)).all()


_TRSM = r"""
import ctypes, sys, numpy as np
sys.path.insert(0, %r)
import oracle, synth
L = ctypes.CDLL(%r)
i = lambda v: ctypes.byref(ctypes.c_int(v))
P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
s, m, n = 6, 150, 37
A = np.asfortranarray(np.tril(synth.uniform(m, m, 1, complex_=True)) * 0.2 + 2 * np.eye(m))
B = np.asfortranarray(synth.uniform(m, n, 2, complex_=True))
B0 = B.copy(order="F")
al = (ctypes.c_double * 2)(0.5, -0.5)
L.ztrsm_(b"L", b"L", b"C", b"N", i(m), i(n), al, P(A), i(m), P(B), i(m))
ok_z = bool((B == oracle.trsm("L", "L", "C", "N", 0.5 - 0.5j, A, B0, s)).all())
Ad = np.asfortranarray(np.triu(synth.uniform(n, n, 3)) * 0.3 + 2 * np.eye(n))
Bd = np.asfortranarray(synth.uniform(m, n, 4))
Bd0 = Bd.copy(order="F")
a1 = ctypes.c_double(1.0)
L.dtrsm_(b"R", b"U", b"N", b"U", i(m), i(n), ctypes.byref(a1), P(Ad), i(n), P(Bd), i(m))
ok_d = bool((Bd == oracle.trsm("R", "U", "N", "U", 1.0, Ad, Bd0, s)).all())
L.dtrsm_(b"R", b"Q", b"N", b"U", i(m), i(n), ctypes.byref(a1), P(Ad), i(n), P(Bd), i(m))
print("OK" if ok_d and ok_z else "MISMATCH", ok_d, ok_z)
"""


@pytest.mark.gpu
def test_shim_trsm_bitexact_vs_oracle(shim):
    """ztrsm_ / dtrsm_ (Fortran ABI, host arrays) = the oracle's R23 blocked TRSM, bit for bit;
    an invalid UPLO gets the xerbla message with parameter number 2."""
    r = _run_py(_TRSM % (ROOT, shim), {"OZAKI_NUM_SLICES": "6"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.startswith("OK"), r.stdout + r.stderr[-2000:]
    assert "On entry to DTRSM  parameter number  2 had an illegal value" in r.stderr
