"""TEST INFRASTRUCTURE -- CPU restatement of the reference solve path.

This module restates, function by function, the algorithm of the reference
package ``fastpoisson`` 0.1.0 (`/root/reference/pkg/src/fastpoisson/`) for the
hot path `SolverPlan.solve` (solver.py:191-249).  It is the checker for the
GPU kernels and the CPU baseline of ``bench.py``; the product never imports it.

Third-party dependency named and pinned: the reference delegates its line
transforms to ``scipy.fft`` (installed here: scipy 1.18.1, DUCC0 backend;
the reference pins only ``scipy>=1.10``, pkg/pyproject.toml:10-13).  The
restatement calls the same scipy entry points the reference calls
(transforms.py:70-77,163,171-172; solver.py:239,245).  Independently of scipy,
``naive_transform`` evaluates the defining sums (transforms.py:3-15,188-229)
and ``makhoul_dct2`` / ``makhoul_dct3`` restate the half-length FFT recipes
the GPU kernels use, so the conventions are pinned without trusting scipy.

Pinning: ``tests/test_oracle_golden.py`` checks this oracle against golden
vectors produced by the reference itself (``tests/golden/make_golden.py``),
against the reference tests' known answers, and against the dense FD2 oracle
(verify.py:81-104).  Parity is therefore pinned, not unpinned.
"""

from __future__ import annotations

import itertools
import math

import numpy as np
from scipy import fft as sfft

PERIODIC, DIRICHLET, NEUMANN = "periodic", "dirichlet", "neumann"
REGULAR, STAGGERED = "regular", "staggered"
SPECTRAL, FD2 = "spectral", "fd2"

__all__ = [
    "PERIODIC", "DIRICHLET", "NEUMANN", "REGULAR", "STAGGERED", "SPECTRAL", "FD2",
    "Axis", "Case", "axis_dx", "axis_points", "eigenvalues", "pair", "backward_scale",
    "null_coeff", "forward_1d", "backward_1d", "naive_transform", "makhoul_dct2",
    "makhoul_dct3", "r1_via_rfft", "r1_inverse_via_irfft", "mr_factors", "mr_perm", "mr_fft", "mr_transform", "staggered_divergence", "staggered_gradient",
    "projection_case", "project_step", "solve", "laplacian", "dense_matrix", "dense_solve", "CONFIGS",
    "config_case", "config_rhs", "relative_l2",
]


class Axis(tuple):
    """(n, length, bc, kind)"""

    def __new__(cls, n, length, bc, kind=REGULAR):
        return tuple.__new__(cls, (int(n), float(length), bc, kind))

    n = property(lambda s: s[0])
    length = property(lambda s: s[1])
    bc = property(lambda s: s[2])
    kind = property(lambda s: s[3])


class Case:
    """A solver configuration: axes, approximation, precision ('double'/'single')."""

    def __init__(self, axes, approx, precision="double"):
        self.axes = tuple(Axis(*a) for a in axes)
        self.approx = approx
        self.precision = precision

    @property
    def shape(self):
        return tuple(a.n for a in self.axes)

    @property
    def dtype(self):
        return np.dtype(np.float64 if self.precision == "double" else np.float32)

    @property
    def singular(self):  # solver.py:116-119
        return all(a.bc != DIRICHLET for a in self.axes)

    @property
    def periodic_axes(self):  # solver.py:105-109
        return tuple(i for i, a in enumerate(self.axes) if a.bc == PERIODIC)


# -- grid.py:80-100 ------------------------------------------------------------
def axis_dx(a: Axis) -> float:
    if a.kind == STAGGERED or a.bc == PERIODIC:
        return a.length / a.n
    if a.bc == DIRICHLET:
        return a.length / (a.n + 1)
    return a.length / (a.n - 1)


def axis_points(a: Axis) -> np.ndarray:
    j = np.arange(a.n, dtype=np.float64)
    if a.kind == STAGGERED:
        return (j + 0.5) * (a.length / a.n)
    if a.bc == PERIODIC:
        return j * (a.length / a.n)
    if a.bc == DIRICHLET:
        return (j + 1.0) * (a.length / (a.n + 1))
    return j * (a.length / (a.n - 1))


# -- eigenvalues.py:51-77 ------------------------------------------------------
def eigenvalues(a: Axis, approx: str) -> np.ndarray:
    k = np.arange(a.n, dtype=np.float64)
    if approx == SPECTRAL:
        if a.bc == PERIODIC:
            return -((2.0 * np.pi * np.minimum(k, a.n - k) / a.length) ** 2)
        if a.bc == DIRICHLET:
            return -((np.pi * (k + 1.0) / a.length) ** 2)
        return -((np.pi * k / a.length) ** 2)
    if a.bc == PERIODIC:
        ang = k * np.pi / a.n
    elif a.bc == DIRICHLET:
        ang = np.pi * (k + 1.0) / (2.0 * (a.n + 1 if a.kind == REGULAR else a.n))
    else:
        ang = np.pi * k / (2.0 * (a.n - 1 if a.kind == REGULAR else a.n))
    return -((2.0 * np.sin(ang) / axis_dx(a)) ** 2)


# -- transforms.py:99-125, 88-96 ----------------------------------------------
def pair(a: Axis):
    if a.bc == PERIODIC:
        return "dft", "idft"
    if a.bc == DIRICHLET:
        return ("dst1", "dst1") if a.kind == REGULAR else ("dst2", "dst3")
    return ("dct1", "dct1") if a.kind == REGULAR else ("dct2", "dct3")


def backward_scale(a: Axis) -> float:
    f = pair(a)[0]
    if f == "dft":
        return 1.0
    if f == "dst1":
        return 1.0 / (2.0 * (a.n + 1))
    if f == "dct1":
        return 1.0 / (2.0 * (a.n - 1))
    return 1.0 / (2.0 * a.n)


def null_coeff(a: Axis) -> float:  # solver.py:58-62
    f = pair(a)[0]
    return {"dft": 1.0, "dct1": 2.0 * (a.n - 1), "dct2": 2.0 * a.n}[f]


_REAL = {"dst1": (sfft.dst, 1), "dst2": (sfft.dst, 2), "dst3": (sfft.dst, 3),
         "dct1": (sfft.dct, 1), "dct2": (sfft.dct, 2), "dct3": (sfft.dct, 3)}


def forward_1d(kind, x, axis=-1, workers=None):
    """TransformPlan.execute_real / execute_complex (transforms.py:157-172)."""
    if kind == "dft":
        return sfft.fft(x, axis=axis, workers=workers) / x.shape[axis]
    if kind == "idft":
        return sfft.ifft(x, axis=axis, workers=workers) * x.shape[axis]
    f, t = _REAL[kind]
    return f(x, type=t, axis=axis, workers=workers)


backward_1d = forward_1d


# -- transforms.py:188-229 (independent of scipy) --------------------------------
def naive_transform(kind: str, line) -> np.ndarray:
    x = np.asarray(line)
    n = x.shape[-1]
    j = np.arange(n)
    k = j[:, None]
    if kind == "dft":
        return (np.exp(-2j * np.pi * k * j / n) / n) @ x.astype(np.complex128)
    if kind == "idft":
        return np.exp(2j * np.pi * k * j / n) @ x.astype(np.complex128)
    if kind == "dst1":
        m = 2.0 * np.sin(np.pi * (j + 1) * (k + 1) / (n + 1))
    elif kind == "dst2":
        m = 2.0 * np.sin(np.pi * (j + 0.5) * (k + 1) / n)
    elif kind == "dst3":
        m = 2.0 * np.sin(np.pi * (j + 1) * (k + 0.5) / n)
        m[:, n - 1] = (-1.0) ** np.arange(n)
    elif kind == "dct1":
        m = 2.0 * np.cos(np.pi * j * k / (n - 1))
        m[:, 0] = 1.0
        m[:, n - 1] = (-1.0) ** np.arange(n)
    elif kind == "dct2":
        m = 2.0 * np.cos(np.pi * (j + 0.5) * k / n)
    elif kind == "dct3":
        m = 2.0 * np.cos(np.pi * j * (k + 0.5) / n)
        m[:, 0] = 1.0
    else:
        raise ValueError(kind)
    return m @ (x.astype(np.complex128) if np.iscomplexobj(x) else x.astype(np.float64))


# -- the half-length FFT recipes of the GPU kernels, restated with numpy.fft ---
def makhoul_dct2(x: np.ndarray) -> np.ndarray:
    """DCT-II via Makhoul reordering + n/2-point complex FFT + untangle + twiddle."""
    n = x.shape[-1]
    M = n // 2
    v = np.concatenate([x[..., 0::2], x[..., 1::2][..., ::-1]], axis=-1)
    z = v[..., 0::2] + 1j * v[..., 1::2]
    Z = np.fft.fft(z, axis=-1)
    k = np.arange(M + 1)
    Zk = Z[..., k % M]
    Zm = np.conj(Z[..., (M - k) % M])
    V = 0.5 * (Zk + Zm) - 0.5j * np.exp(-2j * np.pi * k / n) * (Zk - Zm)
    U = np.exp(-1j * np.pi * k / (2 * n)) * V
    X = np.empty(x.shape, dtype=np.float64)
    X[..., : M + 1] = 2.0 * U.real
    X[..., n - k[1:M]] = -2.0 * U[..., 1:M].imag
    return X


def makhoul_dct3(X: np.ndarray) -> np.ndarray:
    """DCT-III via twiddle + tangle + n/2-point inverse complex FFT + de-interleave."""
    n = X.shape[-1]
    M = n // 2
    k = np.arange(n)
    Xe = np.concatenate([X, np.zeros(X.shape[:-1] + (1,))], axis=-1)
    V = np.exp(1j * np.pi * k / (2 * n)) * (Xe[..., k] - 1j * Xe[..., n - k])
    kk = np.arange(M)
    Vk = V[..., kk]
    Vm = np.conj(V[..., (M - kk) % n])
    Z = (Vk + Vm) + 1j * np.exp(2j * np.pi * kk / n) * (Vk - Vm)
    z = np.fft.ifft(Z, axis=-1) * M
    v = np.empty(X.shape, dtype=np.float64)
    v[..., 0::2] = z.real
    v[..., 1::2] = z.imag
    x = np.empty_like(v)
    x[..., 0::2] = v[..., :M]
    x[..., 1::2] = v[..., M:][..., ::-1]
    return x


def r1_via_rfft(x: np.ndarray, kind: str) -> np.ndarray:
    """DCT-I / DST-I as the real FFT of the even / odd 2M-point extension (the
    recipe of the sm_100a kernels for regular grids; the reference computes them
    with scipy.fft.dct/dst type 1, transforms.py:70-77).

    DCT-I (n = M + 1): z = [x_0..x_M, x_{M-1}..x_1], X_k = Re rfft(z)_k.
    DST-I (n = M - 1): z = [0, x, 0, -reverse(x)],   X_{k-1} = -Im rfft(z)_k.
    """
    if kind == "dct1":
        z = np.concatenate([x, x[..., -2:0:-1]], axis=-1)
        return np.fft.rfft(z, axis=-1).real
    zero = np.zeros(x.shape[:-1] + (1,))
    z = np.concatenate([zero, x, zero, -x[..., ::-1]], axis=-1)
    return -np.fft.rfft(z, axis=-1).imag[..., 1:-1]


def r1_inverse_via_irfft(X: np.ndarray, kind: str) -> np.ndarray:
    """The unnormalised DCT-I / DST-I of X computed as the inverse real FFT of the
    half spectrum (X_k, 0) resp. (0, -X_{k-1}), truncated to n outputs (the
    kernels' inverse / second leg of the fused middle pass)."""
    if kind == "dct1":
        M = X.shape[-1] - 1
        return (np.fft.irfft(X.astype(complex), n=2 * M, axis=-1) * (2 * M))[..., : M + 1]
    M = X.shape[-1] + 1
    S = np.zeros(X.shape[:-1] + (M + 1,), dtype=complex)
    S[..., 1:M] = -1j * X
    return (np.fft.irfft(S, n=2 * M, axis=-1) * (2 * M))[..., 1:M]


# -- the mixed-radix engine's recipes (fp_mr.cu), restated with numpy ---------------
def mr_factors(N: int, max_prime: int = 61):
    """Radices in stage order: 16, 8, 4, 2, then odd primes <= max_prime ([] if none fit)."""
    f, m = [], N
    for r in (16, 8, 4, 2):
        while m % r == 0:
            f.append(r)
            m //= r
    p = 3
    while p <= max_prime and m > 1:
        while m % p == 0:
            f.append(p)
            m //= p
        p += 2
    return f if m == 1 else []


def mr_perm(N: int, fac) -> np.ndarray:
    """Digit-reversed position of input index j for the in-place DIT over `fac`."""
    j = np.arange(N)
    pos = np.zeros(N, dtype=np.int64)
    mult = N
    for R in reversed(fac):
        mult //= R
        pos += (j % R) * mult
        j = j // R
    return pos


def mr_fft(z: np.ndarray, inverse: bool = False) -> np.ndarray:
    """Unnormalised complex FFT of the last axis by the kernel's algorithm: scatter
    into digit-reversed order, then in-place DIT stages (radix R, span L) with
    butterflies over {b L R + k1 + r L} twiddled by W_{LR}^{r k1}."""
    N = z.shape[-1]
    fac = mr_factors(N)
    if not fac:
        raise ValueError(f"FFT length {N} has a prime factor above 61: no mixed-radix plan")
    sgn = 1.0 if inverse else -1.0
    root = np.exp(sgn * 2j * np.pi * np.arange(N) / N)
    w = np.empty(z.shape, dtype=np.complex128)
    w[..., mr_perm(N, fac)] = z
    L = 1
    for R in fac:
        Lq = L * R
        r = np.arange(R)
        W = root[(np.outer(r, r) % R) * (N // R)]
        k1 = np.arange(L)
        tw = root[(np.outer(r, k1) * (N // Lq)) % N]                    # (R, L)
        blk = w.reshape(z.shape[:-1] + (N // Lq, R, L)) * tw
        w = np.einsum("kr,...brl->...bkl", W, blk).reshape(z.shape)
        L = Lq
    return w


def blue_fft(z: np.ndarray, inverse: bool = False) -> np.ndarray:
    """Unnormalised complex DFT of the last axis by Bluestein's algorithm as the
    Bluestein engine runs it (csrc/fp_blue.cu): jk = (j^2 + k^2 - (k-j)^2)/2 turns the
    DFT into Z_k = conj(c_k) sum_j (z_j conj(c_j)) c_{k-j}, c_m = e^{i pi m^2/N}
    (conjugated for the inverse sign), a linear convolution evaluated as a cyclic one
    of length L = the power of two >= max(2N - 1, 16); the chirp angle is reduced
    exactly (m^2 mod 2N) as the plan tables are."""
    N = z.shape[-1]
    m = np.arange(N, dtype=np.int64)
    c = np.exp(1j * np.pi * ((m * m) % (2 * N)) / N)
    if inverse:
        c = np.conj(c)
    L = 16
    while L < 2 * N - 1:
        L *= 2
    h = np.zeros(L, dtype=np.complex128)
    h[:N] = c
    h[L - N + 1:] = c[1:][::-1]
    a = np.zeros(z.shape[:-1] + (L,), dtype=np.complex128)
    a[..., :N] = z * np.conj(c)
    conv = np.fft.ifft(np.fft.fft(a) * np.fft.fft(h))
    return conv[..., :N] * np.conj(c)


def mr_transform(kind: str, x: np.ndarray, fft=None) -> np.ndarray:
    """Unnormalised scipy-type transform of the last axis by the mixed-radix recipes
    (any n: Makhoul for II/III, even/odd extensions for I, full complex FFTs).
    `fft` swaps the complex DFT underneath (blue_fft: the Bluestein engine's)."""
    mr_fft_ = fft or mr_fft
    n = x.shape[-1]
    j = np.arange(n)
    mk = np.where(j % 2 == 0, j // 2, n - 1 - j // 2)           # Makhoul position of x_j
    if kind in ("dct2", "dst2"):
        v = np.empty(x.shape, dtype=np.complex128)
        v[..., mk] = x * ((-1.0) ** j if kind == "dst2" else 1.0)
        V = mr_fft_(v)
        y = 2.0 * (np.exp(-1j * np.pi * j / (2 * n)) * V).real
        return y[..., ::-1] if kind == "dst2" else y
    if kind in ("dct3", "dst3"):
        X = x[..., ::-1] if kind == "dst3" else x
        Xn = np.concatenate([np.zeros(X.shape[:-1] + (1,)), X[..., :0:-1]], axis=-1)   # X_{n-k}, X_n = 0
        W = np.exp(1j * np.pi * j / (2 * n)) * (X - 1j * Xn)
        W[..., 0] = X[..., 0]
        y = mr_fft_(W, inverse=True)[..., mk].real
        return y * (-1.0) ** j if kind == "dst3" else y
    if kind == "dct1":
        z = np.concatenate([x, x[..., -2:0:-1]], axis=-1)
        return mr_fft_(z.astype(np.complex128))[..., :n].real
    if kind == "dst1":
        zero = np.zeros(x.shape[:-1] + (1,))
        z = np.concatenate([zero, x, zero, -x[..., ::-1]], axis=-1)
        return -mr_fft_(z.astype(np.complex128))[..., 1:n + 1].imag
    if kind == "dft":
        return mr_fft_(x.astype(np.complex128)) / n
    if kind == "idft":
        return mr_fft_(x.astype(np.complex128), inverse=True)
    if kind == "rfft":   # real-input DFT, outputs k = 0..n/2 (the plan's kind 100)
        return mr_fft_(x.astype(np.complex128))[..., : n // 2 + 1]
    if kind == "irfft":  # half spectrum -> real, unnormalised (kind 101): x has n//2+1 entries
        raise ValueError("irfft: use blue_irfft(x, n)")
    raise ValueError(kind)


def blue_transform(kind: str, x: np.ndarray) -> np.ndarray:
    """The Bluestein engine's algorithm for every kind (mr_transform's recipes on blue_fft)."""
    return mr_transform(kind, x, fft=blue_fft)


def blue_irfft(X: np.ndarray, n: int, fft=None) -> np.ndarray:
    """Half spectrum (n//2+1 entries) -> n reals, unnormalised (the plan's kind 101):
    Hermitian extension, inverse-sign DFT, real part."""
    fft = fft or blue_fft
    h = n // 2 + 1
    k = np.arange(n)
    src = np.where(k < h, k, n - k)
    z = X[..., src]
    z = np.where(k < h, z, np.conj(z))
    return fft(z.astype(np.complex128), inverse=True).real


# -- flow.py: the projection step around the solve ---------------
def staggered_divergence(u: np.ndarray, w: np.ndarray, lengths, z_walls: bool) -> np.ndarray:
    """Cell-centred divergence of face velocities (flow.py:114-122)."""
    nx, nz = u.shape
    dx, dz = lengths[0] / nx, lengths[1] / nz
    div = (np.roll(u, -1, axis=0) - u) / dx
    if z_walls:
        div += (w[:, 1:] - w[:, :-1]) / dz
    else:
        div += (np.roll(w, -1, axis=1) - w) / dz
    return div


def staggered_gradient(phi: np.ndarray, lengths, z_walls: bool):
    """Face gradient of a cell-centred scalar; wall faces get 0 (flow.py:125-139)."""
    nx, nz = phi.shape
    dx, dz = lengths[0] / nx, lengths[1] / nz
    gx = (phi - np.roll(phi, 1, axis=0)) / dx
    if z_walls:
        gz = np.zeros((nx, nz + 1))
        gz[:, 1:-1] = (phi[:, 1:] - phi[:, :-1]) / dz
    else:
        gz = (phi - np.roll(phi, 1, axis=1)) / dz
    return gx, gz


def projection_case(cells, lengths, z_walls: bool) -> "Case":
    """The flow's pressure plan (flow.py:241-250)."""
    nx, nz = cells
    zax = (nz, lengths[1], NEUMANN, STAGGERED) if z_walls else (nz, lengths[1], PERIODIC)
    return Case([(nx, lengths[0], PERIODIC), zax], FD2)


def project_step(ustar, wstar, scale, lengths, z_walls: bool):
    """One projection of a ProjectionFlow stage (flow.py:290-295) -> (u, w, phi)."""
    case = projection_case(ustar.shape, lengths, z_walls)
    rhs = staggered_divergence(ustar, wstar, lengths, z_walls) / scale
    phi, _ = solve(case, rhs)
    gx, gz = staggered_gradient(phi, lengths, z_walls)
    return ustar - scale * gx, wstar - scale * gz, phi


# -- solver.py:136-249 -----------------------------------------------------------
_EXTENDED_LIMIT = 4096  # solver.py:53
_HAVE_EXTENDED = np.finfo(np.longdouble).eps < np.finfo(np.float64).eps


class OraclePlan:
    """Plan-time half of SolverPlan (solver.py:136-181): the dense combined
    eigenvalues and their inverse (eigenvalues.py:94-114, solver.py:149-159),
    built once; ``solve`` is the per-call half (solver.py:191-249)."""

    def __init__(self, case: Case, workers=None, extended=True):
        self.case = case
        self.workers = workers
        shape = case.shape
        dtype = case.dtype
        work_dtype = dtype
        if extended and math.prod(shape) <= _EXTENDED_LIMIT and _HAVE_EXTENDED and dtype == np.float64:
            work_dtype = np.dtype(np.longdouble)
        self.work_dtype = work_dtype
        d = len(shape)
        lam = np.zeros(shape, dtype=np.float64)
        for ax, a in enumerate(case.axes):
            s = [1] * d
            s[ax] = a.n
            lam += eigenvalues(a, case.approx).reshape(s)
        bscale = math.prod(backward_scale(a) for a in case.axes)
        inv = np.zeros_like(lam)
        np.divide(bscale, lam, out=inv, where=lam != 0.0)
        self.inv = inv.astype(work_dtype)

    def solve(self, rhs):
        """Return (solution, removed_mean) exactly as SolverPlan.solve computes them."""
        case, workers, work_dtype = self.case, self.workers, self.work_dtype
        shape = case.shape
        rhs = np.asarray(rhs)
        if rhs.shape != shape:
            raise ValueError("rhs extents do not match")
        if not np.isfinite(rhs).all():
            raise ValueError("rhs contains non-finite values")
        d = len(shape)
        periodic = case.periodic_axes
        real_axes = tuple(i for i in range(d) if i not in periodic)
        work = np.array(rhs, dtype=work_dtype, copy=True, order="C")
        for ax in real_axes:
            work = forward_1d(pair(case.axes[ax])[0], work, axis=ax, workers=workers)
        if periodic:
            scale = math.prod(shape[ax] for ax in periodic)
            work = sfft.fftn(work, axes=periodic, workers=workers) / scale
        removed_mean = 0.0
        if case.singular:
            null_scale = math.prod(null_coeff(a) for a in case.axes)
            removed_mean = float(np.real(work[(0,) * d])) / null_scale
        work *= self.inv
        if periodic:
            scale = math.prod(shape[ax] for ax in periodic)
            work = sfft.ifftn(work, axes=periodic, workers=workers) * scale
            work = np.ascontiguousarray(work.real, dtype=work_dtype)
        for ax in reversed(real_axes):
            work = backward_1d(pair(case.axes[ax])[1], work, axis=ax, workers=workers)
        if case.singular:
            work -= work.mean()
        return np.asarray(work, dtype=case.dtype), removed_mean


def solve(case: Case, rhs, workers=None, extended=True):
    """Return (solution, removed_mean) exactly as SolverPlan.solve computes them
    (plan and solve in one call; see OraclePlan)."""
    rhs = np.asarray(rhs)
    if rhs.shape != case.shape:
        raise ValueError("rhs extents do not match")
    return OraclePlan(case, workers, extended).solve(rhs)


# -- solver.py:286-338 -----------------------------------------------------------
def laplacian(case: Case, field) -> np.ndarray:
    x = np.asarray(field, dtype=np.float64)
    out = np.zeros(x.shape)
    for ax, a in enumerate(case.axes):
        y = np.moveaxis(x, ax, 0)
        r = np.empty_like(y)
        if a.n == 1:
            if a.bc == DIRICHLET:
                r[0] = (-4.0 if a.kind == STAGGERED else -2.0) * y[0]
            else:
                r[0] = 0.0
        else:
            r[1:-1] = y[2:] - 2.0 * y[1:-1] + y[:-2]
            if a.bc == PERIODIC:
                r[0] = y[1] - 2.0 * y[0] + y[-1]
                r[-1] = y[0] - 2.0 * y[-1] + y[-2]
            elif a.bc == DIRICHLET:
                c = -2.0 if a.kind == REGULAR else -3.0
                r[0] = y[1] + c * y[0]
                r[-1] = y[-2] + c * y[-1]
            elif a.kind == REGULAR:
                r[0] = 2.0 * y[1] - 2.0 * y[0]
                r[-1] = 2.0 * y[-2] - 2.0 * y[-1]
            else:
                r[0] = y[1] - y[0]
                r[-1] = y[-2] - y[-1]
        r /= axis_dx(a) ** 2
        out += np.moveaxis(r, 0, ax)
    return out


# -- verify.py:29-104 --------------------------------------------------------------
def _stencil(a: Axis) -> np.ndarray:
    n = a.n
    m = np.zeros((n, n))
    i = np.arange(n)
    m[i, i] = -2.0
    m[i[:-1], i[:-1] + 1] = 1.0
    m[i[1:], i[1:] - 1] = 1.0
    if a.bc == PERIODIC:
        if n == 1:
            m[0, 0] = 0.0
        else:
            m[0, -1] += 1.0
            m[-1, 0] += 1.0
    elif a.bc == DIRICHLET:
        if a.kind == STAGGERED:
            m[0, 0] = m[-1, -1] = -3.0 if n > 1 else -4.0
    elif a.kind == REGULAR:
        m[0, 1] = 2.0
        m[-1, -2] = 2.0
    else:
        m[0, 0] = m[-1, -1] = -1.0 if n > 1 else 0.0
    return m / axis_dx(a) ** 2


def dense_matrix(case: Case) -> np.ndarray:
    mats = [_stencil(a) for a in case.axes]
    total = math.prod(case.shape)
    out = np.zeros((total, total))
    for ax, m in enumerate(mats):
        term = np.ones((1, 1))
        for j, a in enumerate(case.axes):
            term = np.kron(term, m if j == ax else np.eye(a.n))
        out += term
    return out


def dense_solve(case: Case, rhs) -> np.ndarray:
    import scipy.linalg

    g = np.asarray(rhs, dtype=np.float64).ravel()
    mat = dense_matrix(case)
    if not case.singular:
        return np.linalg.solve(mat, g).reshape(case.shape)
    w = scipy.linalg.null_space(mat.T)[:, 0]
    g = g - (w @ g) / w.sum()
    sol = np.linalg.lstsq(mat, g, rcond=None)[0]
    sol -= sol.mean()
    return sol.reshape(case.shape)


def relative_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b.ravel())
    return float(np.linalg.norm((a - b).ravel()) / (den if den > 0 else 1.0))


# -- BASELINE.json configs and their seeded right-hand sides -----
TWO_PI = 2.0 * np.pi
CONFIGS = {
    "c1": Case([(64, TWO_PI, PERIODIC)] * 3, SPECTRAL),
    "c2": Case([(4096, 1.0, DIRICHLET, STAGGERED)] * 2, FD2),
    "c3": Case([(512, 1.0, NEUMANN, STAGGERED)] * 3, FD2),
    "c4": Case([(1024, TWO_PI, PERIODIC), (1024, TWO_PI, PERIODIC), (512, 2.0, NEUMANN, STAGGERED)], FD2),
    "c5": Case([(2048, TWO_PI, PERIODIC)] * 3, SPECTRAL, "single"),
}


def config_case(name: str, scale: int = 1) -> Case:
    """The named config, optionally with every axis divided by ``scale``."""
    c = CONFIGS[name]
    if scale == 1:
        return c
    return Case([(a.n // scale, a.length, a.bc, a.kind) for a in c.axes], c.approx, c.precision)


def config_rhs(name: str, case: Case, seed: int = 0) -> np.ndarray:
    """Seeded RHS with the distribution BASELINE.json names for the config."""
    rng = np.random.default_rng(seed)
    shape = case.shape
    if name in ("c1", "c3"):
        r = rng.standard_normal(shape)
        return r - r.mean()
    if name == "c2":
        x = axis_points(case.axes[0])
        y = axis_points(case.axes[1])
        return rng.standard_normal(shape) + np.sin(np.pi * x)[:, None] * np.sin(np.pi * y)[None, :]
    if name == "c4":
        nx, ny, nz = shape
        dx = axis_dx(case.axes[0])
        dy = axis_dx(case.axes[1])
        dz = axis_dx(case.axes[2])
        u = rng.standard_normal(shape)
        v = rng.standard_normal(shape)
        w = rng.standard_normal((nx, ny, nz + 1))
        w[..., 0] = 0.0
        w[..., -1] = 0.0
        return ((np.roll(u, -1, 0) - u) / dx + (np.roll(v, -1, 1) - v) / dy + (w[..., 1:] - w[..., :-1]) / dz)
    if name == "c5":
        r = rng.standard_normal(shape, dtype=np.float32)
        r -= np.float32(r.astype(np.float64).mean())
        return r
    raise KeyError(name)
