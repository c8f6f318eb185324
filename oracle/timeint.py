"""TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference integrators
(hybridwave/timeint.py) plus the 2N-storage LSRK(4,5) of Carpenter &
Kennedy (NASA TM-109112, 1994), which the reference does not contain.

``rhs`` arguments are callables ``rhs(state, time) -> dict``.
"""

import math

import numpy as np

# Carpenter-Kennedy (4,5) 2N-storage coefficients
LSRK_A = [0.0,
          -567301805773.0 / 1357537059087.0,
          -2404267990393.0 / 2016746695238.0,
          -3550918686646.0 / 2091501179385.0,
          -1275806237668.0 / 842570457699.0]
LSRK_B = [1432997174477.0 / 9575080441755.0,
          5161836677717.0 / 13612068292357.0,
          1720146321549.0 / 2090206949498.0,
          3134564353537.0 / 4481467310338.0,
          2277821191437.0 / 14882151754819.0]
LSRK_C = [0.0,
          1432997174477.0 / 9575080441755.0,
          2526269341429.0 / 6820363962896.0,
          2006345519317.0 / 3224310063776.0,
          2802321613138.0 / 2924317926251.0]


def ab_coefficients(n_hist, theta=1.0):
    """hybridwave/timeint.py:21-38."""
    th = theta
    if n_hist == 1:
        return np.array([th])
    if n_hist == 2:
        return np.array([th + th ** 2 / 2.0, -(th ** 2) / 2.0])
    if n_hist == 3:
        return np.array([th + 3.0 * th ** 2 / 4.0 + th ** 3 / 6.0,
                         -(th ** 2) - th ** 3 / 3.0,
                         th ** 2 / 4.0 + th ** 3 / 6.0])
    raise ValueError("history depth must be 1..3")


def ab3_step(state, history, dt, theta=1.0):
    """hybridwave/timeint.py:41-54."""
    c = ab_coefficients(len(history), theta)
    out = {}
    for t, a in state.items():
        acc = np.array(a, copy=True)
        for ci, f in zip(c, history):
            acc += dt * ci * f[t]
        out[t] = acc
    return out


def single_rate_run(rhs, state, dt, T_final, callback=None):
    """hybridwave/timeint.py:57-72."""
    time, hist = 0.0, []
    while time < T_final - 1e-14:
        h = min(dt, T_final - time)
        hist.insert(0, rhs(state, time))
        del hist[3:]
        state = ab3_step(state, hist, dt, theta=h / dt)
        time += h
        if callback is not None:
            callback(time, state)
    return state


def lsrk_run(rhs, state, dt, T_final, callback=None):
    """5-stage 2N-storage RK: res = a_i res + h rhs(q, t + c_i h);
    q += b_i res.  Final step shortened to land on T_final."""
    q = {t: np.array(v, copy=True) for t, v in state.items()}
    res = {t: np.zeros_like(v) for t, v in q.items()}
    time = 0.0
    while time < T_final - 1e-14:
        h = min(dt, T_final - time)
        for a, bcoef, c in zip(LSRK_A, LSRK_B, LSRK_C):
            k = rhs(q, time + c * h)
            for t in q:
                res[t] = a * res[t] + h * k[t]
                q[t] = q[t] + bcoef * res[t]
        time += h
        if callback is not None:
            callback(time, q)
    return q


def mrab_run(rhs, levels, n_levels, dt_min, state, T_final, callback=None):
    """Multi-rate AB3 (hybridwave/timeint.py:75-173).  ``levels`` is a dict
    t -> (K,) ints in 1..n_levels (level 1 coarsest); ``dt_min`` the plan's
    finest step.  Mutates and returns ``state`` and the per-type RHS
    evaluation counts."""
    L = n_levels
    macro = 2 ** (L - 1) * dt_min
    n_macro = max(1, math.ceil(T_final / macro - 1e-12))
    dt_min = T_final / (n_macro * 2 ** (L - 1))
    masks = {t: [levels[t] == lev for lev in range(1, L + 1)] for t in state}
    hist = {t: np.zeros((3,) + state[t].shape) for t in state}
    n_hist = np.zeros(L + 1, dtype=int)
    evals = {t: np.zeros(len(levels[t]), dtype=int) for t in state}
    for m in range(n_macro):
        t0 = m * dt_min * 2 ** (L - 1)
        for tick in range(2 ** (L - 1)):
            stepping = [lev for lev in range(1, L + 1) if tick % (2 ** (L - lev)) == 0]
            tau = t0 + tick * dt_min
            eff = {}
            for t in state:
                e = state[t].copy()
                for lev in range(1, L + 1):
                    period = 2 ** (L - lev)
                    frac = tick % period
                    sel = masks[t][lev - 1]
                    if frac == 0 or n_hist[lev] == 0 or not sel.any():
                        continue
                    nh = n_hist[lev]
                    c = ab_coefficients(nh, frac / period) - ab_coefficients(nh, 1.0)
                    upd = sum(c[i] * hist[t][i, sel] for i in range(nh))
                    e[sel] += dt_min * period * upd
                eff[t] = e
            r = rhs(eff, tau)
            for t in state:
                sel = np.zeros(len(levels[t]), dtype=bool)
                for lev in stepping:
                    sel |= masks[t][lev - 1]
                if not sel.any():
                    continue
                evals[t][sel] += 1
                hist[t][2, sel] = hist[t][1, sel]
                hist[t][1, sel] = hist[t][0, sel]
                hist[t][0, sel] = r[t][sel]
            for lev in stepping:
                n_hist[lev] = min(n_hist[lev] + 1, 3)
                dt_lev = dt_min * 2 ** (L - lev)
                c = ab_coefficients(n_hist[lev])
                for t in state:
                    sel = masks[t][lev - 1]
                    if not sel.any():
                        continue
                    upd = c[0] * hist[t][0, sel]
                    for i in range(1, n_hist[lev]):
                        upd += c[i] * hist[t][i, sel]
                    state[t][sel] += dt_lev * upd
        if callback is not None:
            callback(t0 + dt_min * 2 ** (L - 1), state)
    return state, evals
