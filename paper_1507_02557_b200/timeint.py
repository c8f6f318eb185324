"""Device-resident time integration behind the reference's timeint API
(hybridwave/timeint.py:17-181) plus LSRK-45.

Every step is one fused kernel launch per element type (RHS + update); the
state, residual and Adams-Bashforth history live in HBM for the whole run.
``single_rate_run`` / ``lsrk_run`` / ``mrab_run`` accept numpy states (the
reference's host arrays: copied in once, out at the end and for callbacks)
or CUDA tensors (stay on the device).
"""

import math

import numpy as np
import torch

from . import _native as nat
from .operators import TYPE_ID

__all__ = ["ab_coefficients", "ab3_step", "single_rate_run", "MRABDriver", "mrab_run",
           "lsrk_step", "lsrk_run", "LSRK_A", "LSRK_B", "LSRK_C", "Stepper"]

# Carpenter & Kennedy (1994) (4,5) 2N-storage
LSRK_A = (0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
          -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0)
LSRK_B = (1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
          1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
          2277821191437.0 / 14882151754819.0)
LSRK_C = (0.0, 1432997174477.0 / 9575080441755.0, 2526269341429.0 / 6820363962896.0,
          2006345519317.0 / 3224310063776.0, 2802321613138.0 / 2924317926251.0)


def ab_coefficients(n_hist, theta=1.0):
    """u(t + theta h) = u(t) + h sum c_i f_i (hybridwave/timeint.py:21-38)."""
    th = theta
    if n_hist == 1:
        return np.array([th])
    if n_hist == 2:
        return np.array([th + th ** 2 / 2.0, -(th ** 2) / 2.0])
    if n_hist == 3:
        return np.array([th + 3.0 * th ** 2 / 4.0 + th ** 3 / 6.0, -(th ** 2) - th ** 3 / 3.0,
                         th ** 2 / 4.0 + th ** 3 / 6.0])
    raise ValueError("history depth must be 1..3")


def ab3_step(state, history, dt, theta=1.0):
    """hybridwave/timeint.py:41-54 (numpy or torch dicts)."""
    c = ab_coefficients(len(history), theta)
    out = {}
    for t, a in state.items():
        acc = a.clone() if isinstance(a, torch.Tensor) else np.array(a, copy=True)
        for ci, f in zip(c, history):
            acc += dt * float(ci) * f[t]
        out[t] = acc
    return out


def _is_host(state):
    return not isinstance(next(iter(state.values())), torch.Tensor)


def _export(disc, q, host, out=None):
    """Device state -> the caller's side: new host arrays, or (out given)
    written into the caller's host arrays (pinned ones copy at DMA speed)."""
    if host and out is not None:
        for t in disc.types:
            torch.from_numpy(out[t]).copy_(q[t])
        return out
    if host:
        return {t: q[t].cpu().numpy() for t in disc.types}
    return {t: q[t].clone() for t in disc.types}


def _no_forcing(disc):
    if disc.forcing is not None:
        raise NotImplementedError("lsrk_step takes no forcing callback; use lsrk_run")


class Stepper:
    """Device buffers and launch sequence for one integrator, reusable by
    the benchmark (and CUDA-graph capturable: no host syncs, fixed
    pointers when ``swap=False``)."""

    def __init__(self, disc, state, scheme="lsrk"):
        self.disc = disc
        self.dm = disc.device_mesh
        self.q = disc.to_device(state)
        self.q2 = disc.empty_state()
        self.scheme = scheme
        if scheme == "lsrk":
            self.res = disc.zeros_state()
        else:
            self.hist = [disc.zeros_state() for _ in range(3)]
            self.n_steps = 0
        self.launches_per_stage = len(disc.types)
        # traces of the initial state; stages then ping-pong the trace sets
        self.tr = 0
        self.dm.compute_traces(self._f(self.q), 0, disc.stream_ptr())

    def _stage_traces(self):
        self.dm.set_traces(self.tr, 1 - self.tr)
        self.tr = 1 - self.tr

    def _f(self, s):
        return nat.fields(self.disc.slots(s))

    def lsrk_step(self, h, time=0.0):
        """One LSRK(4,5) step from `time`.  With a forcing callback, each
        stage's forcing term (at time + c_i h) is integrated on the device
        (hw_forcing) and added in the stage kernel's epilogue."""
        L = nat.lib()
        st = self.disc.stream_ptr()
        extra = False
        for a, b, c in zip(LSRK_A, LSRK_B, LSRK_C):
            self._stage_traces()
            extra = self.disc.prepare_stage(time + c * h) or extra
            nat.check(L.hw_lsrk_stage(self.dm.struct, self._f(self.q), self._f(self.q2),
                                      self._f(self.res), a, b, h, None, st))
            self.q, self.q2 = self.q2, self.q
        if extra:
            self.disc.clear_forcing()

    def ab_step(self, dt, theta=1.0, time=0.0):
        nh = min(self.n_steps + 1, 3)
        c = ab_coefficients(nh, theta)
        c = list(c) + [0.0] * (3 - len(c))
        new = self.hist[2]
        self._stage_traces()
        extra = self.disc.prepare_stage(time)
        nat.check(nat.lib().hw_ab_step(self.dm.struct, self._f(self.q), self._f(self.q2),
                                       self._f(new), self._f(self.hist[0]),
                                       self._f(self.hist[1]), nh, c[0], c[1], c[2], dt, None,
                                       self.disc.stream_ptr()))
        if extra:
            self.disc.clear_forcing()
        self.hist = [new, self.hist[0], self.hist[1]]
        self.q, self.q2 = self.q2, self.q
        self.n_steps += 1


def _view(disc, q, host):
    """State handed to a callback: the live device buffers for a device run
    (the reference also passes live references, timeint.py:68-70; no
    copy, no sync), fresh host arrays for a host run."""
    return _export(disc, q, True) if host else dict(q)


def _want_callback(callback, every, n, time, T_final):
    return callback is not None and (n % every == 0 or time >= T_final - 1e-14)


def single_rate_run(disc, state, dt, T_final, callback=None, out=None, callback_every=1):
    """AB3 to T_final; the last step lands through the fractional
    coefficients (hybridwave/timeint.py:57-72).  out: optional host arrays
    the final state is written into; callback_every: call back every k-th
    step (and after the last).  A forcing callback is integrated on the
    device each step and added in the fused kernel's epilogue."""
    host = _is_host(state)
    S = Stepper(disc, state, "ab")
    time, n = 0.0, 0
    while time < T_final - 1e-14:
        h = min(dt, T_final - time)
        S.ab_step(dt, theta=h / dt, time=time)
        time += h
        n += 1
        if _want_callback(callback, callback_every, n, time, T_final):
            callback(time, _view(disc, S.q, host))
    return _export(disc, S.q, host, out)


def lsrk_step(disc, q, res, dt, q_tmp=None):
    """One 5-stage LSRK(4,5) step on device dicts (q, res updated; q is
    returned, possibly a different buffer set when q_tmp is supplied)."""
    _no_forcing(disc)
    dm = disc.device_mesh
    q_tmp = q_tmp if q_tmp is not None else disc.empty_state()
    st = disc.stream_ptr()
    dm.compute_traces(nat.fields(disc.slots(q)), 0, st)
    tr = 0
    for a, b in zip(LSRK_A, LSRK_B):
        dm.set_traces(tr, 1 - tr)
        tr = 1 - tr
        if dm.corr:
            disc.apply_corrections()
        nat.check(nat.lib().hw_lsrk_stage(dm.struct, nat.fields(disc.slots(q)),
                                          nat.fields(disc.slots(q_tmp)),
                                          nat.fields(disc.slots(res)), a, b, dt, None, st))
        q, q_tmp = q_tmp, q
    disc.clear_forcing()
    return q


def lsrk_run(disc, state, dt, T_final, callback=None, out=None, callback_every=1):
    """Low-storage RK(4,5) to T_final with the single_rate_run signature;
    the last step is shortened to land on T_final."""
    host = _is_host(state)
    S = Stepper(disc, state, "lsrk")
    time, n = 0.0, 0
    while time < T_final - 1e-14:
        h = min(dt, T_final - time)
        S.lsrk_step(h, time=time)
        time += h
        n += 1
        if _want_callback(callback, callback_every, n, time, T_final):
            callback(time, _view(disc, S.q, host))
    return _export(disc, S.q, host, out)


class MRABDriver:
    """Multi-rate AB3 (hybridwave/timeint.py:75-173) that launches only the
    active levels: each tick evaluates the RHS of the stepping elements
    alone (the reference evaluates the whole mesh and discards the rest),
    fused with their AB update; coarse neighbours are seen through their
    dense-output extrapolation.  Same arithmetic for every consumed entry."""

    def __init__(self, disc, plan):
        self.disc = disc
        self.plan = plan
        plan.validate_neighbor_levels(disc.mesh)
        self.levels = {t: plan.levels_of(disc.mesh, t) for t in disc.types}
        self.n_levels = plan.n_levels
        self.rhs_evals = {t: np.zeros(disc.n_elems[t], dtype=int) for t in disc.types}
        self.macro_steps = 0
        dev = disc.device
        # element lists per level per type (int32 on the device)
        self._lists = {}
        for lev in range(1, self.n_levels + 1):
            for t in disc.types:
                idx = np.flatnonzero(self.levels[t] == lev).astype(np.int32)
                self._lists[(lev, t)] = torch.as_tensor(idx, device=dev) if len(idx) else None
        self._tick_subsets()

    def _tick_subsets(self):
        """Per tick of the macro step: the elements whose effective state and
        face traces the stepping elements read (themselves and their face
        neighbours), so the dense-output pass and the trace pass touch only
        those instead of the whole mesh."""
        disc, L = self.disc, self.n_levels
        mesh = disc.mesh
        names = ("hex", "wedge", "pyramid", "tet")
        need = {lev: {t: self.levels[t] == lev for t in disc.types} for lev in range(1, L + 1)}
        for lev in range(1, L + 1):
            own = {t: need[lev][t].copy() for t in disc.types}
            for t in disc.types:
                nb = mesh.nbr[t][own[t]]                       # (n, nf, 3)
                for tid2, t2 in enumerate(names):
                    if t2 not in need[lev]:
                        continue
                    sel = nb[:, :, 0] == tid2
                    need[lev][t2][nb[:, :, 1][sel]] = True
        dev = disc.device
        empty = torch.zeros(0, dtype=torch.int32, device=dev)
        self._tick_keep, self._eff_subs, self._trace_subs = [], {}, {}
        for tick in range(2 ** (L - 1)):
            stepping = [lev for lev in range(1, L + 1) if tick % (2 ** (L - lev)) == 0]
            needed = {t: np.any([need[lev][t] for lev in stepping], axis=0) for t in disc.types}
            tl = [None] * 4
            for t in disc.types:
                idx = np.flatnonzero(needed[t]).astype(np.int32)
                tl[TYPE_ID[t]] = torch.as_tensor(idx, device=dev) if len(idx) else empty
            self._tick_keep.append(tl)
            self._trace_subs[tick] = nat.subset(tl)
            for lev in range(1, L + 1):
                el = [None] * 4
                any_ = False
                for t in disc.types:
                    idx = np.flatnonzero(needed[t] & (self.levels[t] == lev)).astype(np.int32)
                    el[TYPE_ID[t]] = torch.as_tensor(idx, device=dev) if len(idx) else empty
                    any_ |= len(idx) > 0
                for t in range(4):
                    if el[t] is None:
                        el[t] = empty
                self._tick_keep.append(el)
                self._eff_subs[(tick, lev)] = nat.subset(el) if any_ else None

    def _subset(self, levs):
        lists = [None] * 4
        empty = torch.zeros(0, dtype=torch.int32, device=self.disc.device)
        for t in self.disc.types:
            parts = [self._lists[(lev, t)] for lev in levs if self._lists[(lev, t)] is not None]
            lists[TYPE_ID[t]] = torch.cat(parts) if parts else empty
        return lists

    def _macro(self, q, eff, ring, n_hist, steps, dt_min, st):
        """Launch one macro step (2^(L-1) ticks) on stream st; advances the
        host-side counters n_hist / steps / rhs_evals.  Returns (q, eff):
        tick 0 steps every level, so it reads q directly and writes the new
        state into the other buffer (no effective-state copy of the whole
        mesh); the two buffers swap roles once per macro step."""
        disc, L = self.disc, self.n_levels
        lib, dm = nat.lib(), disc.device_mesh
        F = lambda s: nat.fields(disc.slots(s))
        subs = self._sub_structs
        for tick in range(2 ** (L - 1)):
            stepping = [lev for lev in range(1, L + 1) if tick % (2 ** (L - lev)) == 0]
            if tick == 0:   # every level steps: q is the effective state everywhere
                dm.compute_traces(F(q), 0, st, subset=self._trace_subs[tick])
                dm.set_traces(0, None)
                if dm.corr:
                    disc.apply_corrections()
                for lev in stepping:
                    n_hist[lev] = min(n_hist[lev] + 1, 3)
                    steps[lev] += 1
                    s0 = steps[lev] % 3
                    h0, h1, h2 = ring[s0], ring[(s0 - 1) % 3], ring[(s0 - 2) % 3]
                    nh = n_hist[lev]
                    c = list(ab_coefficients(nh)) + [0.0] * (3 - nh)
                    nat.check(lib.hw_ab_step(dm.struct, F(q), F(eff), F(h0), F(h1), F(h2), nh,
                                             c[0], c[1], c[2], dt_min * 2 ** (L - lev),
                                             subs[lev], st))
                q, eff = eff, q
                continue
            # effective state: q, plus the dense-output correction on
            # non-stepping levels (timeint.py:144-173)
            for lev in range(1, L + 1):
                period = 2 ** (L - lev)
                frac = tick % period
                nh = n_hist[lev]
                sub = self._eff_subs[(tick, lev)]        # read by this tick's stepping elements
                if sub is None:
                    continue
                if frac == 0 or nh == 0:
                    nat.check(lib.hw_axpy3(dm.struct, F(q), F(eff), F(ring[0]), None, None,
                                           1, 0.0, 0.0, 0.0, 0.0, sub, st))
                    continue
                c = ab_coefficients(nh, frac / period) - ab_coefficients(nh, 1.0)
                c = list(c) + [0.0] * (3 - nh)
                s0 = steps[lev] % 3
                h = [ring[s0], ring[(s0 - 1) % 3], ring[(s0 - 2) % 3]]
                nat.check(lib.hw_axpy3(dm.struct, F(q), F(eff), F(h[0]), F(h[1]), F(h[2]),
                                       nh, c[0], c[1], c[2], dt_min * period, sub, st))
            # traces of the effective state, then the fused RHS + AB update
            # of each stepping level (no trace publishing)
            dm.compute_traces(F(eff), 0, st, subset=self._trace_subs[tick])
            dm.set_traces(0, None)
            if dm.corr:
                disc.apply_corrections()
            for lev in stepping:
                n_hist[lev] = min(n_hist[lev] + 1, 3)
                steps[lev] += 1
                s0 = steps[lev] % 3
                h0, h1, h2 = ring[s0], ring[(s0 - 1) % 3], ring[(s0 - 2) % 3]
                nh = n_hist[lev]
                c = list(ab_coefficients(nh)) + [0.0] * (3 - nh)
                nat.check(lib.hw_ab_step(dm.struct, F(eff), F(q), F(h0), F(h1), F(h2), nh,
                                         c[0], c[1], c[2], dt_min * 2 ** (L - lev),
                                         subs[lev], st))
        self._count(1)
        return q, eff

    def _count(self, n_macro):
        L = self.n_levels
        for t in self.disc.types:
            for lev in range(1, L + 1):
                self.rhs_evals[t][self.levels[t] == lev] += n_macro * 2 ** (lev - 1)

    def _run_forced(self, state, T_final, callback):
        """With a forcing callback: per tick the full-mesh RHS of the
        effective state plus the forcing at the tick time (unfused, host
        forcing), then the history push and AB3 update of the stepping
        levels, in the reference's order (hybridwave/timeint.py:111-142)."""
        disc, L = self.disc, self.n_levels
        host = _is_host(state)
        macro = 2 ** (L - 1) * self.plan.dt_min
        n_macro = max(1, math.ceil(T_final / macro - 1e-12))
        dt_min = T_final / (n_macro * 2 ** (L - 1))
        q = disc.to_device(state)
        hist = {t: torch.zeros((3,) + tuple(q[t].shape), dtype=q[t].dtype, device=q[t].device)
                for t in disc.types}
        n_hist = np.zeros(L + 1, dtype=int)
        masks = {t: [torch.as_tensor(self.levels[t] == lev, device=q[t].device)
                     for lev in range(1, L + 1)] for t in disc.types}
        for m in range(n_macro):
            t0 = m * dt_min * 2 ** (L - 1)
            for tick in range(2 ** (L - 1)):
                stepping = [lev for lev in range(1, L + 1) if tick % (2 ** (L - lev)) == 0]
                eff = {}
                for t in disc.types:
                    e = q[t].clone()
                    for lev in range(1, L + 1):
                        period = 2 ** (L - lev)
                        frac = tick % period
                        nh = n_hist[lev]
                        if frac == 0 or nh == 0:
                            continue
                        c = ab_coefficients(nh, frac / period) - ab_coefficients(nh, 1.0)
                        sel = masks[t][lev - 1]
                        upd = float(c[0]) * hist[t][0][sel]
                        for i in range(1, nh):
                            upd = upd + float(c[i]) * hist[t][i][sel]
                        e[sel] += dt_min * period * upd
                    eff[t] = e
                rhs = disc.rhs_device(eff)
                disc._add_forcing(rhs, t0 + tick * dt_min)
                for t in disc.types:
                    sel = torch.zeros_like(masks[t][0])
                    for lev in stepping:
                        sel |= masks[t][lev - 1]
                    if not bool(sel.any()):
                        continue
                    self.rhs_evals[t][sel.cpu().numpy()] += 1
                    hist[t][2][sel] = hist[t][1][sel]
                    hist[t][1][sel] = hist[t][0][sel]
                    hist[t][0][sel] = rhs[t][sel]
                for lev in stepping:
                    n_hist[lev] = min(n_hist[lev] + 1, 3)
                    c = ab_coefficients(n_hist[lev])
                    for t in disc.types:
                        sel = masks[t][lev - 1]
                        upd = float(c[0]) * hist[t][0][sel]
                        for i in range(1, n_hist[lev]):
                            upd = upd + float(c[i]) * hist[t][i][sel]
                        q[t][sel] += dt_min * 2 ** (L - lev) * upd
            self.macro_steps += 1
            if callback is not None:
                callback(t0 + dt_min * 2 ** (L - 1), _view(disc, q, host))
        out = _export(disc, q, host)
        for t in disc.types:
            if host:
                state[t][...] = out[t]
            else:
                state[t].copy_(out[t])
        return state

    def run(self, state, T_final, callback=None, graph=True):
        """graph: once every level holds 3 history entries the launch
        pattern repeats every 3 macro steps (ring slots cycle mod 3); that
        period is captured once as a CUDA graph and replayed (no callback).
        A forcing callback takes the unfused path (_run_forced)."""
        if self.disc.forcing is not None:
            return self._run_forced(state, T_final, callback)
        disc = self.disc
        L = self.n_levels
        host = _is_host(state)
        macro = 2 ** (L - 1) * self.plan.dt_min
        n_macro = max(1, math.ceil(T_final / macro - 1e-12))
        dt_min = T_final / (n_macro * 2 ** (L - 1))
        if getattr(self, "_bufs", None) is None:      # persistent work buffers
            # the driver owns the state buffers it steps (the caller's
            # state is copied in and written back at the end), so a captured
            # graph's pointers stay valid for every later run()
            self._bufs = (disc.empty_state(), [disc.zeros_state() for _ in range(3)],
                          disc.empty_state())
            subs = {lev: self._subset([lev]) for lev in range(1, L + 1)}
            self._subs_keep = subs
            self._sub_structs = {lev: nat.subset(subs[lev]) for lev in subs}
            self._graphs = {}
        eff, ring, q = self._bufs
        src = disc.to_device(state)
        for t in disc.types:
            q[t].copy_(src[t])
        del src
        n_hist = np.zeros(L + 1, dtype=int)
        steps = np.zeros(L + 1, dtype=int)
        use_graph = graph and callback is None
        m = 0
        while m < n_macro:
            t0 = m * dt_min * 2 ** (L - 1)
            if use_graph and n_macro - m >= 3 and (n_hist[1:] == 3).all():
                # the period's graph depends on which buffer holds q (the
                # buffers swap once per macro step, an odd number per period)
                gkey = (dt_min, q[disc.types[0]].data_ptr())
                g = self._graphs.get(gkey)
                if g is None:
                    g = self._graphs[gkey] = torch.cuda.CUDAGraph()
                    saved = (n_hist.copy(), steps.copy(), {t: v.copy() for t, v in self.rhs_evals.items()})
                    qq, ee = q, eff
                    with torch.cuda.graph(g):
                        for _ in range(3):
                            qq, ee = self._macro(qq, ee, ring, n_hist, steps, dt_min,
                                                 disc.stream_ptr())
                    # capture launches nothing: restore the counters, replay below
                    n_hist[:], steps[:] = saved[0], saved[1]
                    self.rhs_evals = saved[2]
                g.replay()
                q, eff = eff, q
                for lev in range(1, L + 1):
                    steps[lev] += 3 * 2 ** (lev - 1)
                self._count(3)
                self.macro_steps += 3
                m += 3
                continue
            q, eff = self._macro(q, eff, ring, n_hist, steps, dt_min, disc.stream_ptr())
            self.macro_steps += 1
            m += 1
            if callback is not None:
                callback(t0 + dt_min * 2 ** (L - 1), _view(disc, q, host))
        out = _export(disc, q, host)
        for t in disc.types:
            if host:
                state[t][...] = out[t]
            else:
                state[t].copy_(out[t])
        return state


def mrab_run(disc, plan, state, T_final, callback=None):
    """hybridwave/timeint.py:176-181: returns (state, driver); state is
    updated in place like the reference's."""
    driver = MRABDriver(disc, plan)
    driver.run(state, T_final, callback=callback)
    return state, driver
