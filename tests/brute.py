"""Independent brute-force re-derivations used to pin the oracle.

None of this calls or mirrors oracle/pic_oracle.c's code paths:
* gather: sum over ALL nodes of minimum-image linear hats (no floor/i0 logic);
* current: exact Gauss-Legendre integration of the plain flux definition
  J_x dt = qw int_0^1 dX 1[floor x(tau) = i] S(y(tau)-j) S(z(tau)-k) dtau / (dy dz)
  (SURVEY.md sec. 8c O5 "plain definition") -- no segment splitting or
  Villasenor-Buneman weight formulas;
* curls: numpy FFT symbols of forward / backward differences.
"""
from __future__ import annotations

import numpy as np

STAG = np.array([[0.5, 0, 0], [0, 0.5, 0], [0, 0, 0.5],
                 [0, 0.5, 0.5], [0.5, 0, 0.5], [0.5, 0.5, 0]])


def min_image(d, n):
    return (d + n / 2.0) % n - n / 2.0


def hat(xi):
    return np.maximum(0.0, 1.0 - np.abs(xi))


def hat_gather(F6, h, pos):
    """F6: (6, nz, ny, nx); h = (dx,dy,dz); pos physical (3,)."""
    nz, ny, nx = F6.shape[1:]
    g = np.asarray(pos, dtype=np.float64) / np.asarray(h)
    out = np.zeros(6)
    for c in range(6):
        o = STAG[c]
        sx = hat(min_image(g[0] - o[0] - np.arange(nx), nx))
        sy = hat(min_image(g[1] - o[1] - np.arange(ny), ny))
        sz = hat(min_image(g[2] - o[2] - np.arange(nz), nz))
        out[c] = np.einsum("k,j,i,kji->", sz, sy, sx, F6[c])
    return out


_GL_X, _GL_W = np.polynomial.legendre.leggauss(4)


def flux_current(shape, h, dt, qw, a_phys, b_phys):
    """Exact integral of the CIC-cloud flux for the straight move a -> b.

    Returns J (3, nz, ny, nx).  Breakpoints are every tau where some
    coordinate crosses an integer; between them the integrand is a
    polynomial of degree <= 2, so 4-point Gauss-Legendre is exact."""
    nz, ny, nx = shape
    n = (nx, ny, nz)
    h = np.asarray(h, dtype=np.float64)
    a = np.asarray(a_phys, dtype=np.float64) / h
    b = np.asarray(b_phys, dtype=np.float64) / h
    D = b - a
    taus = [0.0, 1.0]
    for d in range(3):
        if D[d] != 0:
            lo, hi = min(a[d], b[d]), max(a[d], b[d])
            for m in range(int(np.floor(lo)) - 1, int(np.floor(hi)) + 2):
                t = (m - a[d]) / D[d]
                if 0.0 < t < 1.0:
                    taus.append(t)
    taus = np.unique(np.array(taus))
    J = np.zeros((3, nz, ny, nx))
    scale = [qw / (dt * h[1] * h[2]), qw / (dt * h[0] * h[2]), qw / (dt * h[0] * h[1])]
    for t0, t1 in zip(taus[:-1], taus[1:]):
        if t1 <= t0:
            continue
        for xg, wg in zip(_GL_X, _GL_W):
            t = 0.5 * (t0 + t1) + 0.5 * (t1 - t0) * xg
            wt = 0.5 * (t1 - t0) * wg
            p = a + t * D
            fl = np.floor(p).astype(np.int64)
            fr = p - fl
            for d in range(3):
                e1, e2 = [e for e in range(3) if e != d]
                for s1 in (0, 1):
                    for s2 in (0, 1):
                        w1 = fr[e1] if s1 else 1.0 - fr[e1]
                        w2 = fr[e2] if s2 else 1.0 - fr[e2]
                        idx = [0, 0, 0]
                        idx[d] = fl[d] % n[d]
                        idx[e1] = (fl[e1] + s1) % n[e1]
                        idx[e2] = (fl[e2] + s2) % n[e2]
                        J[d, idx[2], idx[1], idx[0]] += scale[d] * D[d] * wt * w1 * w2
    return J


def rho_hat(shape, h, qw, pos_list):
    """Node charge density by brute-force hats over all nodes."""
    nz, ny, nx = shape
    g_h = np.asarray(h, dtype=np.float64)
    rho = np.zeros(shape)
    V = g_h.prod()
    for pos in pos_list:
        g = np.asarray(pos) / g_h
        sx = hat(min_image(g[0] - np.arange(nx), nx))
        sy = hat(min_image(g[1] - np.arange(ny), ny))
        sz = hat(min_image(g[2] - np.arange(nz), nz))
        rho += qw / V * np.einsum("k,j,i->kji", sz, sy, sx)
    return rho


def _diff_fft(f, axis, hx, forward):
    n = f.shape[axis]
    m = np.fft.fftfreq(n) * n
    ph = np.exp(2j * np.pi * m / n)
    sym = (ph - 1.0) / hx if forward else (1.0 - 1.0 / ph) / hx
    shape = [1, 1, 1]
    shape[axis] = n
    return np.real(np.fft.ifft(np.fft.fft(f, axis=axis) * sym.reshape(shape), axis=axis))


# array axes: (z, y, x) -> axis index for physical axis d is 2 - d
def dfwd(f, d, h):
    return _diff_fft(f, 2 - d, h[d], True)


def dbwd(f, d, h):
    return _diff_fft(f, 2 - d, h[d], False)


def fft_b_half(F, h, c, dt):
    Ex, Ey, Ez = F[0], F[1], F[2]
    cx = dfwd(Ez, 1, h) - dfwd(Ey, 2, h)
    cy = dfwd(Ex, 2, h) - dfwd(Ez, 0, h)
    cz = dfwd(Ey, 0, h) - dfwd(Ex, 1, h)
    G = F.copy()
    G[3] -= 0.5 * c * dt * cx
    G[4] -= 0.5 * c * dt * cy
    G[5] -= 0.5 * c * dt * cz
    return G


def fft_e_full(F, h, c, dt):
    Bx, By, Bz = F[3], F[4], F[5]
    cx = dbwd(Bz, 1, h) - dbwd(By, 2, h)
    cy = dbwd(Bx, 2, h) - dbwd(Bz, 0, h)
    cz = dbwd(By, 0, h) - dbwd(Bx, 1, h)
    G = F.copy()
    G[0] += c * dt * cx - 4 * np.pi * dt * F[6]
    G[1] += c * dt * cy - 4 * np.pi * dt * F[7]
    G[2] += c * dt * cz - 4 * np.pi * dt * F[8]
    return G


def boris_np(q, m, c, dt, EB, u):
    h = q * dt / (2 * m * c)
    E, B = np.asarray(EB[:3]), np.asarray(EB[3:])
    um = u + h * E
    t = h * B / np.sqrt(1 + um @ um)
    up = um + np.cross(um, t)
    upl = um + np.cross(up, t) * (2 / (1 + t @ t))
    return upl + h * E


def brute_step(F, parts, species, h, c, dt):
    """One full PIC step with the brute-force pieces (O2 order)."""
    nz, ny, nx = F.shape[1:]
    L = np.array([nx, ny, nz]) * np.asarray(h)
    F = F.copy()
    F[6:] = 0.0
    new_parts = []
    for (q, m, w), P in zip(species, parts):
        P = P.copy()
        for p in range(P.shape[1]):
            x = P[:3, p].copy()
            EB = hat_gather(F[:6], h, x)
            u = boris_np(q, m, c, dt, EB, P[3:, p])
            xn = x + dt * c * u / np.sqrt(1 + u @ u)
            F[6:] += flux_current((nz, ny, nx), h, dt, q * w, x, xn)
            P[:3, p] = np.mod(xn, L)
            P[3:, p] = u
        new_parts.append(P)
    F = fft_b_half(F, h, c, dt)
    F = fft_e_full(F, h, c, dt)
    F = fft_b_half(F, h, c, dt)
    return F, new_parts
