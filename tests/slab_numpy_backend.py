"""numpy restatement of the three slab kernel groups of libsrk (TEST INFRASTRUCTURE).

Same buffer layouts as csrc/srk_api.cu srk_slab_forward / _middle / _finish:
  send1/recv1 [rank][s][x_loc][y_loc][kz], send2/recv2 [rank][o][x_loc][y_loc][kz].
Used by tests/test_slab_gloo.py to exercise paper_1810_10197_b200.slab on CPU
(gloo, world_size > 1) against the single-process oracle RHS.
"""
import numpy as np
import torch

from paper_1810_10197_b200.slab import slab_geometry


def _modes_full(n):
    m = np.arange(n, dtype=np.float64)
    m[m > n // 2] -= n
    return m


class NumpySlabBackend:
    def __init__(self, grid, params, rank, nranks, density=False):
        self.g = slab_geometry(grid, nranks, density)
        self.rank, self.P, self.density = rank, nranks, density
        self.params = params
        L = grid.lengths
        g = self.g
        self.kx = (_modes_full(g["n0"]) * (2 * np.pi / L[0]))[:, None, None]
        ky_all = _modes_full(g["n1"]) * (2 * np.pi / L[1])
        self.ky_full = ky_all
        self.ky = ky_all[rank * g["ny"]:(rank + 1) * g["ny"]][None, :, None]
        self.kz = (np.arange(g["K"], dtype=np.float64) * (2 * np.pi / L[2]))[None, None, :]
        self.scale_in = 1.5 ** 3 / (g["m0"] * g["m1"] * g["m2"])

    def empty(self, n):
        return torch.empty(n, dtype=torch.complex128)

    @staticmethod
    def _pad(a, axis, n, m):
        shp = list(a.shape)
        shp[axis] = m
        out = np.zeros(shp, dtype=np.complex128)
        h = [slice(None)] * a.ndim
        t_s = [slice(None)] * a.ndim
        t_d = [slice(None)] * a.ndim
        h[axis] = slice(0, n // 2 + 1)
        t_s[axis] = slice(n // 2 + 1, n)
        t_d[axis] = slice(m - (n // 2 - 1), m)
        out[tuple(h)] = a[tuple(h)]
        out[tuple(t_d)] = a[tuple(t_s)]
        return out

    @staticmethod
    def _trunc(a, axis, n, m):
        shp = list(a.shape)
        shp[axis] = n
        out = np.zeros(shp, dtype=np.complex128)
        h = [slice(None)] * a.ndim
        t_s = [slice(None)] * a.ndim
        t_d = [slice(None)] * a.ndim
        h[axis] = slice(0, n // 2)
        t_s[axis] = slice(m - (n // 2 - 1), m)
        t_d[axis] = slice(n // 2 + 1, n)
        out[tuple(h)] = a[tuple(h)]
        out[tuple(t_d)] = a[tuple(t_s)]
        return out

    def forward(self, y, send1):
        g, u = self.g, y.numpy()
        kx, ky, kz = self.kx, self.ky, self.kz
        sig = [u[0], u[1], u[2], kx * u[1], kx * u[2]]  # curl completed in middle()
        if self.density:
            sig.append(u[3])
        out = send1.numpy().reshape(self.P, g["S1"], g["mx"], g["ny"], g["K"])
        for s, a in enumerate(sig):
            p = np.fft.ifft(self._pad(a * self.scale_in, 0, g["n0"], g["m0"]), axis=0) * g["m0"]
            for d in range(self.P):
                out[d, s] = p[d * g["mx"]:(d + 1) * g["mx"]]

    def middle(self, recv1, send2):
        g = self.g
        r = recv1.numpy().reshape(self.P, g["S1"], g["mx"], g["ny"], g["K"])
        w1 = np.concatenate([r[q] for q in range(self.P)], axis=2)  # (S1, mx, n1, K)
        kyf = (self.ky_full)[None, :, None]
        kz = self.kz
        U0, U1, U2, X1, X2 = w1[0], w1[1], w1[2], w1[3], w1[4]
        sig = [U0, U1, U2, 1j * (kyf * U2 - kz * U1), 1j * (kz * U0 - X2), 1j * (X1 - kyf * U0)]
        if self.density:
            sig.append(w1[5])
        full = np.stack(sig)
        a = np.fft.ifft(self._pad(full, 2, g["n1"], g["m1"]), axis=2) * g["m1"]
        ph = np.fft.irfft(a, n=g["m2"], axis=3) * g["m2"]
        u, w = ph[:3], ph[3:6]
        prods = [u[1] * w[2] - u[2] * w[1], u[2] * w[0] - u[0] * w[2], u[0] * w[1] - u[1] * w[0]]
        if self.density:
            prods += [ph[6] * u[0], ph[6] * u[1], ph[6] * u[2]]
        sp = np.fft.rfft(np.stack(prods), axis=3)[..., : g["K"]]
        sp[..., g["K"] - 1] = 0.0
        t = self._trunc(np.fft.fft(sp, axis=2), 2, g["n1"], g["m1"])  # (So, mx, n1, K), Nyquist row 0
        out = send2.numpy().reshape(self.P, g["So"], g["mx"], g["ny"], g["K"])
        for d in range(self.P):
            out[d] = t[:, :, d * g["ny"]:(d + 1) * g["ny"]]

    def finish(self, recv2, y, f):
        g = self.g
        r = recv2.numpy().reshape(self.P, g["So"], g["mx"], g["ny"], g["K"])
        full = np.concatenate([r[q] for q in range(self.P)], axis=1)  # (So, m0, ny, K)
        G = self._trunc(np.fft.fft(full, axis=1), 1, g["n0"], g["m0"]) * (1.0 / 1.5) ** 3
        if self.rank == 0:
            G[:, 0, 0, 0] = G[:, 0, 0, 0].real
        self._project(G, y, f)

    # ---- kz-chunked groups (same layouts as srk_slab_*_kz) ----
    def forward_kz(self, y, send1_c, k0, kc):
        g, u = self.g, y.numpy()[..., k0:k0 + kc]
        kx = self.kx
        sig = [u[0], u[1], u[2], kx * u[1], kx * u[2]]
        if self.density:
            sig.append(u[3])
        out = send1_c.numpy().reshape(self.P, g["S1"], g["mx"], g["ny"], kc)
        for s, a in enumerate(sig):
            p = np.fft.ifft(self._pad(a * self.scale_in, 0, g["n0"], g["m0"]), axis=0) * g["m0"]
            for d in range(self.P):
                out[d, s] = p[d * g["mx"]:(d + 1) * g["mx"]]

    def inverse_y_kz(self, recv1_c, k0, kc):
        g = self.g
        if not hasattr(self, "B"):
            self.B = np.zeros((g["S"], g["mx"], g["m1"], g["K"]), dtype=np.complex128)
        r = recv1_c.numpy().reshape(self.P, g["S1"], g["mx"], g["ny"], kc)
        w1 = np.concatenate([r[q] for q in range(self.P)], axis=2)  # (S1, mx, n1, kc)
        kyf = (self.ky_full)[None, :, None]
        kz = self.kz[..., k0:k0 + kc]
        U0, U1, U2, X1, X2 = w1[0], w1[1], w1[2], w1[3], w1[4]
        sig = [U0, U1, U2, 1j * (kyf * U2 - kz * U1), 1j * (kz * U0 - X2), 1j * (X1 - kyf * U0)]
        if self.density:
            sig.append(w1[5])
        self.B[..., k0:k0 + kc] = np.fft.ifft(self._pad(np.stack(sig), 2, g["n1"], g["m1"]), axis=2) * g["m1"]

    def zpass(self):
        g = self.g
        ph = np.fft.irfft(self.B, n=g["m2"], axis=3) * g["m2"]
        u, w = ph[:3], ph[3:6]
        prods = [u[1] * w[2] - u[2] * w[1], u[2] * w[0] - u[0] * w[2], u[0] * w[1] - u[1] * w[0]]
        if self.density:
            prods += [ph[6] * u[0], ph[6] * u[1], ph[6] * u[2]]
        sp = np.fft.rfft(np.stack(prods), axis=3)[..., : g["K"]]
        sp[..., g["K"] - 1] = 0.0
        self.A = sp

    def forward_y_kz(self, send2_c, k0, kc):
        g = self.g
        t = self._trunc(np.fft.fft(self.A[..., k0:k0 + kc], axis=2), 2, g["n1"], g["m1"])
        out = send2_c.numpy().reshape(self.P, g["So"], g["mx"], g["ny"], kc)
        for d in range(self.P):
            out[d] = t[:, :, d * g["ny"]:(d + 1) * g["ny"]]

    def forward_x_kz(self, recv2_c, k0, kc):
        g = self.g
        if not hasattr(self, "G"):
            self.G = np.zeros((g["So"], g["n0"], g["ny"], g["K"]), dtype=np.complex128)
        r = recv2_c.numpy().reshape(self.P, g["So"], g["mx"], g["ny"], kc)
        full = np.concatenate([r[q] for q in range(self.P)], axis=1)  # (So, m0, ny, kc)
        G = self._trunc(np.fft.fft(full, axis=1), 1, g["n0"], g["m0"]) * (1.0 / 1.5) ** 3
        if self.rank == 0 and k0 == 0:
            G[:, 0, 0, 0] = G[:, 0, 0, 0].real
        self.G[..., k0:k0 + kc] = G

    def project(self, y, f):
        self._project(self.G, y, f)

    def _project(self, G, y, f):
        g, p = self.g, self.params
        u = y.numpy()
        k = (self.kx, self.ky, self.kz)
        k2 = (0 + k[0] * k[0]) + k[1] * k[1] + k[2] * k[2]
        inv = np.where(k2 == 0, 0.0, 1.0 / np.where(k2 == 0, 1.0, k2))
        out = f.numpy()
        if self.density:
            G[2] = G[2] - p.richardson * u[3]
        kd = (k[0] * G[0] + k[1] * G[1] + k[2] * G[2]) * inv
        nu = 1.0 / p.reynolds
        for j in range(3):
            out[j] = G[j] - k[j] * kd - (nu * k2) * u[j]
        if self.density:
            div = k[0] * G[3] + k[1] * G[4] + k[2] * G[5]
            out[3] = -1j * div - (k2 / (p.reynolds * p.prandtl)) * u[3]
