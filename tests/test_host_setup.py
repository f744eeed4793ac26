"""CPU: the product's C++ host setup (libkronop.so, no GPU needed) against the oracle, and the
C-ABI library surface: it loads without a GPU and exports every symbol include/kronop_cuda.h
declares."""
import os
import re

import numpy as np
import pytest

from oracle import kronop_oracle as K

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def api():
    from paper_2605_20491_b200 import api as a
    return a


def header_symbols():
    with open(os.path.join(ROOT, "include", "kronop_cuda.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kronop_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2605_20491_b200 import _lib
    h = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(h, s)]
    assert not missing, missing
    # the Python binding declares a prototype for every exported entry point
    assert set(syms) == set(_lib.PROTOTYPES), set(syms) ^ set(_lib.PROTOTYPES)
    assert b"sm_100a" in _lib.lib().kronop_version()


def test_library_is_sm100a_cubin():
    import subprocess
    from paper_2605_20491_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _lib.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "mode_product_kernel" in sass
    assert "DMMA" in sass  # FP64 tensor-core MMA in the transform kernel
    assert "LDGSTS" in sass  # cp.async producer pipeline


@pytest.mark.parametrize("k", [1, 2, 3, 5, 8, 10, 20, 25, 40])
def test_gll_rule_bitwise(k):
    x, w, d = api().gll_rule(k)
    r = K.gll_rule(k)
    assert np.array_equal(x, r.nodes) and np.array_equal(w, r.weights)
    assert np.abs(d - r.diff).max() == 0.0


def test_gauss_legendre_bitwise():
    for m in range(1, 17):
        x, w = api().gauss_legendre(m)
        ox, ow = K.gauss_legendre(m)
        assert np.array_equal(x, ox) and np.array_equal(w, ow)


@pytest.mark.parametrize("spec", [(8.0, 13, 5), (1.0, 16, 2), (8.0, 8, 10), (8.0, 2, 20), (5.0, 3, 10)])
def test_assemble_sem_bitwise(spec):
    b = api().assemble_sem(*spec)
    ob = K.assemble_sem(*spec)
    assert np.array_equal(b.nodes, ob.nodes)
    assert np.array_equal(b.mass, ob.mass)
    assert np.array_equal(b.stiffness, ob.stiffness)


def test_interp_matrix_bitwise():
    A = api()
    for (c, f) in [((8.0, 2, 20), (8.0, 4, 20)), ((8.0, 2, 10), (8.0, 3, 10)), ((1.0, 3, 2), (1.0, 7, 2))]:
        p = A.interp_matrix(A.assemble_sem(*c), A.assemble_sem(*f))
        op = K.interp_matrix(K.assemble_sem(*c), K.assemble_sem(*f))
        assert np.array_equal(p, op)
        assert np.all(p.sum(axis=1) <= 1.0 + 1e-15) and np.all(p >= 0)


@pytest.mark.parametrize("n", [1, 2, 5, 33, 128])
def test_sym_eig_against_lapack(n):
    a = K.uniform_pm1(n, n * n).reshape(n, n)
    a = a + a.T
    lam, q = api().sym_eig(a)
    olam, oq = K.sym_eig(a)
    scale = np.abs(olam).max()
    assert np.abs(lam - olam).max() < 1e-13 * scale * max(1, n / 10)
    assert np.abs(q.T @ q - np.eye(n)).max() < 1e-13 * max(1, n / 10)
    assert np.abs(q @ np.diag(lam) @ q.T - a).max() < 1e-13 * scale * max(1, n / 10)
    # sign convention (axis.cpp:44-52)
    for j in range(n):
        col = q[:, j]
        i = int(np.argmax(np.abs(col) >= (1 - 1e-8) * np.abs(col).max()))
        assert col[i] > 0


def test_sym_eig_analytic_tridiagonal():
    # test_axis_eigen.cpp:42-58: tridiag(-1, 2, -1) has eigenvalues 2 - 2 cos(j pi / (n+1))
    n = 50
    a = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    lam, _ = api().sym_eig(a)
    exact = 2 - 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1))
    assert np.abs(lam - np.sort(exact)).max() < 1e-13
    from paper_2605_20491_b200 import ParameterError
    with pytest.raises(ParameterError):
        api().sym_eig(np.array([[1.0, 2.0], [0.0, 1.0]]))


@pytest.mark.parametrize("spec,f", [((8.0, 13, 5), lambda t: t * t),
                                    ((1.0, 8, 10), lambda t: 1600 * np.sin(np.pi * t / 4) ** 2 + 2 * t * t),
                                    ((8.0, 2, 20), lambda t: 4 * t * t)])
def test_build_axis_factorisation(spec, f):
    """T diag(L) T^-1 is the axis operator M^-1 S + diag(f) (axis.cpp:55-74); eigenvalues equal
    the oracle's; T T^-1 = I. (Eigenvectors of (near-)degenerate pairs are not unique, so T is
    compared through the operator it factorises.)"""
    A = api()
    b = A.assemble_sem(*spec)
    ax = A.build_axis(b, f)
    ob = K.assemble_sem(*spec)
    oax = K.build_axis(ob, f)
    scale = np.abs(oax.eigenvalues).max()
    assert np.abs(ax.eigenvalues - oax.eigenvalues).max() < 1e-12 * scale
    n = b.size
    assert np.abs(ax.transform @ ax.inverse_transform - np.eye(n)).max() < 1e-11
    dense = K.dense_axis_operator(ob, f)
    rec = ax.transform @ np.diag(ax.eigenvalues) @ ax.inverse_transform
    assert np.abs(rec - dense).max() < 1e-11 * scale


def test_host_error_codes():
    from paper_2605_20491_b200 import ParameterError
    A = api()
    with pytest.raises(ParameterError):
        A.gll_rule(0)
    with pytest.raises(ParameterError):
        A.gauss_legendre(17)
    with pytest.raises(ParameterError):
        A.assemble_sem(-1.0, 3, 2)


def _unfold_rows(fa):
    """Full-length T^-1 (rows = modes in folded order) and T (columns) from the folded blocks."""
    n, ne, no = fa.n, len(fa.eigenvalues_even), len(fa.eigenvalues_odd)
    ti = np.zeros((n, n))
    t = np.zeros((n, n))
    for i in range(no):
        ti[:ne, i] = fa.fe[:, i]
        ti[:ne, n - 1 - i] = fa.fe[:, i]
        ti[ne:, i] = fa.fo[:, i]
        ti[ne:, n - 1 - i] = -fa.fo[:, i]
        t[i, :ne] = fa.be[i, :]
        t[n - 1 - i, :ne] = fa.be[i, :]
        t[i, ne:] = fa.bo[i, :]
        t[n - 1 - i, ne:] = -fa.bo[i, :]
    if n % 2:
        ti[:ne, no] = fa.fe[:, no]
        t[no, :ne] = fa.be[no, :]
    return t, ti


@pytest.mark.parametrize("spec,f", [((8.0, 4, 7), lambda t: t * t),          # n = 29 (odd)
                                    ((8.0, 3, 5), lambda t: t * t),          # n = 16 (even)
                                    ((1.0, 8, 10), lambda t: 1600 * np.sin(np.pi * t / 4) ** 2 + 2 * t * t),
                                    ((2.0, 1, 3), None),                     # n = 2
                                    ((2.0, 1, 2), lambda t: 3.0)])           # n = 1
def test_build_axis_folded_reassembles_full_factorisation(spec, f):
    """The even/odd blocks reassemble a factorisation T diag(L) T^-1 of the same axis operator;
    the eigenvalues (sorted) equal the unfolded ones and the mode vectors agree with build_axis's
    (same sign rule) wherever the eigenvalue is simple."""
    A = api()
    b = A.assemble_sem(*spec)
    fa = A.build_axis_folded(b, f)
    ax = A.build_axis(b, f)
    n = b.size
    lam = fa.eigenvalues
    scale = max(np.abs(ax.eigenvalues).max(), 1.0)
    assert np.abs(np.sort(lam) - ax.eigenvalues).max() < 1e-12 * scale
    t, ti = _unfold_rows(fa)
    assert np.abs(t @ ti - np.eye(n)).max() < 1e-11
    dense = K.dense_axis_operator(K.assemble_sem(*spec), f or (lambda x: 0.0))
    assert np.abs(t @ np.diag(lam) @ ti - dense).max() < 1e-11 * scale
    order = np.argsort(lam, kind="stable")
    gaps = np.diff(ax.eigenvalues)
    for r, k in enumerate(order):
        lo = gaps[r - 1] if r > 0 else np.inf
        hi = gaps[r] if r < n - 1 else np.inf
        if min(lo, hi) > 1e-6 * scale:
            assert np.abs(ti[k] - ax.inverse_transform[r]).max() < 1e-9 * np.abs(ti[k]).max()
    assert np.abs(fa.ground - ax.transform[:, 0]).max() < 1e-10 * np.abs(fa.ground).max()


def test_build_axis_folded_rejects_asymmetric_potential():
    from paper_2605_20491_b200 import ParameterError
    A = api()
    b = A.assemble_sem(2.0, 3, 4)
    with pytest.raises(ParameterError):
        A.build_axis_folded(b, lambda t: t * t + 0.1 * t)



@pytest.mark.parametrize("n", [2, 3, 20, 40, 99, 200])
def test_hermite_basis_and_axis_against_oracle(n):
    """hermite_basis / build_axis(HermiteBasis) (hermite.cpp:10-95, axis.cpp:76-84) in the C++
    host setup against the oracle: nodes, psi_{n-1}, mass and D to rounding; eigenvalues to
    1e-12; the factorisation reproduces the dense operator."""
    A = api()
    b = A.hermite_basis(n)
    ob = K.hermite_basis(n)
    assert np.abs(b.nodes - ob.nodes).max() <= 1e-13 * max(1.0, np.abs(ob.nodes).max())
    assert np.array_equal(b.nodes, -b.nodes[::-1])
    assert np.abs(b.psi_last - ob.psi_last).max() <= 1e-10 * np.abs(ob.psi_last).max()
    assert np.abs(b.mass / ob.mass - 1.0).max() <= 1e-10
    assert np.abs(b.diff - ob.diff).max() <= 1e-10 * np.abs(ob.diff).max()
    f = lambda x: x * x + 0.5 * np.cos(x)
    ax = A.build_axis(b, f)
    oax = K.build_hermite_axis(ob, f)
    scale = np.abs(oax.eigenvalues).max()
    assert np.abs(ax.eigenvalues - oax.eigenvalues).max() <= 1e-12 * scale
    assert np.abs(ax.transform @ ax.inverse_transform - np.eye(n)).max() < 1e-10
    dense = K.dense_hermite_axis_operator(ob, f)
    rec = ax.transform @ np.diag(ax.eigenvalues) @ ax.inverse_transform
    assert np.abs(rec - dense).max() < 1e-9 * np.abs(dense).max()


def test_hermite_error_codes():
    from paper_2605_20491_b200 import ParameterError, CapabilityError
    A = api()
    with pytest.raises(ParameterError):
        A.hermite_basis(1)
    with pytest.raises(CapabilityError):
        A.hermite_basis(746)
    with pytest.raises(ParameterError):
        A.build_axis(A.hermite_basis(5), lambda x: float("inf"))


def test_field_io_host_round_trip_and_oracle_format(tmp_path):
    """dump_field / load_field (fieldio.cpp:28-73) through the C-ABI host entry points: the
    product's files load in the oracle's restatement of the reference reader and vice versa,
    bit for bit, for real and complex fields; the reference's error cases raise ParameterError."""
    from paper_2605_20491_b200 import ParameterError
    A = api()
    shape = (5, 3, 4)
    x = K.uniform_pm1(5, 60)
    z = K.seeded_complex_field(shape, 6)
    for data in (x, z):
        p1, p2 = str(tmp_path / "a.kf"), str(tmp_path / "b.kf")
        A.dump_field(p1, data, shape)
        got, shp = K.load_field(p1)
        assert shp == shape and np.array_equal(got, data)
        K.dump_field(p2, data, shape)
        back, shp2, cplx = A.load_field(p2)
        assert shp2 == shape and cplx == np.iscomplexobj(data) and np.array_equal(back, data)
        assert open(p1, "rb").read() == open(p2, "rb").read()
    bad = tmp_path / "bad.kf"
    raw = bytearray(open(str(tmp_path / "a.kf"), "rb").read())
    for mutate, msg in ((lambda r: r.__setitem__(slice(0, 4), b"XXXX"), "bad magic"),
                        (lambda r: r.__setitem__(slice(4, 8), (2).to_bytes(4, "little")), "bad version"),
                        (lambda r: r.__setitem__(slice(8, 12), (10).to_bytes(4, "little")), "bad dimension"),
                        (lambda r: r.__setitem__(slice(12, 16), (7).to_bytes(4, "little")), "unknown scalar kind")):
        r = bytearray(raw)
        mutate(r)
        bad.write_bytes(bytes(r))
        with pytest.raises(ParameterError, match=msg):
            A.load_field(str(bad))
        with pytest.raises(K.ParameterError, match=msg):
            K.load_field(str(bad))
    bad.write_bytes(bytes(raw[:-8]))
    with pytest.raises(ParameterError, match="truncated"):
        A.load_field(str(bad))
    with pytest.raises(ParameterError, match="cannot open"):
        A.load_field(str(tmp_path / "missing.kf"))
