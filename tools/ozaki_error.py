"""Error of the fixed-point rounding that the INT8-CRT R formation (rint8.cu) makes, on darc rows
(300 channels x all 40000 poles of BASELINE.json:10), at mesh energies and at energies 1e-3 / 1e-5
from isolated poles: X = W diag(1/(E_k - E)) and W are rounded to b-bit integers per row (relative to
the row maximum) and the resulting R error dX W^T + X dW^T is measured normwise against R. Prints
the worst error and the number of 8-bit moduli the CRT needs for that b (2b + log2(nlev) + 1 bits).

    PYTHONPATH=. python tools/ozaki_error.py
"""
import numpy as np

import rmx_synth as syn

c = syn.make_case("darc", ne=64)
w = c.w[:300]
Ek = c.Ek
rng = np.random.default_rng(1)
E = list(c.E[::8])
for k in rng.choice(np.where((Ek > 1) & (Ek < 59))[0], 6, replace=False):
    E += [Ek[k] + 1e-3, Ek[k] - 1e-5]
for b in (40, 44, 48, 52):
    worst = 0.0
    for e in E:
        d = 1.0 / (Ek - e)
        X = w * d[None, :]
        sx = np.floor(np.log2(np.max(np.abs(X), axis=1)))
        sw = np.floor(np.log2(np.max(np.abs(w), axis=1)))
        Xs = X * 2.0 ** (b - 1 - sx)[:, None]
        Ws = w * 2.0 ** (b - 1 - sw)[:, None]
        dX = (np.rint(Xs) - Xs) * 2.0 ** (sx - b + 1)[:, None]
        dW = (np.rint(Ws) - Ws) * 2.0 ** (sw - b + 1)[:, None]
        R = X @ w.T
        Err = dX @ w.T + X @ dW.T
        worst = max(worst, np.max(np.abs(Err)) / np.max(np.abs(R)))
    print(b, f"{worst:.2e}", "moduli needed:", int(np.ceil((2 * b + np.log2(40000) + 1) / 7.85)))
