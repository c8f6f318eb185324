"""Drop-in ``Discretization`` whose right-hand side runs on the sm_100a
kernels (reference interface: hybridwave/dg.py:89-572).

Same constructor, same state layout (dict type -> (K, 4, Np)), same entry
points (``compute_rhs``, ``apply_A``, ``compute_traces``,
``apply_mass_inverse``, ``project``, ``eval_at``, ``l2_error``,
``state_to_vector``/``vector_to_state``) and attributes (``types``,
``n_elems``, ``ops``, ``data``, ``n_dof``, ``trace_size``, ``gather_idx``,
``bnd_mask``, ``dof_base``).  States may be numpy arrays (host buffers:
copied to HBM and back inside the call, like the reference's fresh output
arrays) or CUDA tensors (stay resident; the fast path).

``compute_rhs`` has no CPU fallback: without the native library or a GPU it
raises.  The reference-layout arrays (``data``, ``gather_idx`` …) are built
lazily on the host for the diagnostics and the test oracle; the kernels use
the compact layout of ``device.py``.
"""

import numpy as np
import torch

from . import basis as bas
from . import _native as nat
from .operators import TYPE_ID, build_operators, face_symmetry_perms
from .quadrature import element_rule
from .refelem import (FACES, duffy_map, face_geometry_batch, geometric_factors_batch,
                      inverse_duffy_map, jacobian_det, jacobian_det_fast, map_points)

__all__ = ["Formulation", "TABLE_FORMS", "flux_penalties", "Discretization",
           "discrete_energy", "zero_state", "FIELDS"]

TABLE_FORMS = {
    "SEM": {"tet": "strong", "pyramid": "skew", "wedge": "skew", "hex": "strong"},
    "GL": {"tet": "strong", "pyramid": "strong", "wedge": "skew", "hex": "strong"},
}
FIELDS = 4


class Formulation:
    """SEM or GL with the per-type forms of the stability table
    (hybridwave/dg.py:42-58)."""

    def __init__(self, kind):
        if kind not in TABLE_FORMS:
            raise ValueError(f"formulation must be 'SEM' or 'GL', got {kind!r}")
        self.kind = kind
        self.forms = dict(TABLE_FORMS[kind])

    def form(self, elem_type):
        return self.forms[elem_type]

    def __repr__(self):
        return f"Formulation({self.kind!r})"


def flux_penalties(rho_m, c_m, rho_p, c_p):
    """(tau_p, tau_u) = (1/avg(rho c), avg(rho c)) (hybridwave/dg.py:61-69)."""
    if min(rho_m, c_m, rho_p, c_p) <= 0:
        raise ValueError("material parameters must be positive")
    avg = 0.5 * (rho_m * c_m + rho_p * c_p)
    return 1.0 / avg, avg


def zero_state(disc):
    return {t: np.zeros((disc.n_elems[t], FIELDS, disc.ops[t].Np)) for t in disc.types}


class _TypeData:
    """Reference-layout per-type data (hybridwave/dg.py:77-86), host numpy."""

    def __init__(self):
        self.w3 = None
        self.gJfac = None
        self.J_row = None
        self.x_nodes = None
        self.invsqrtJ_face = None
        self.cub_sqrtJ = None
        self.over_sqrtJ = None


def _default_device():
    return torch.device("cuda") if torch.cuda.is_available() else None


class Discretization:
    """Operators, geometry and coupling for one mesh / order / formulation."""

    def __init__(self, mesh, N, formulation, forms_override=None, penalty_scale=1.0,
                 forcing=None, *, dtype=torch.float64, device=None):
        if isinstance(formulation, str):
            formulation = Formulation(formulation)
        self.mesh = mesh
        self.N = N
        self.formulation = formulation
        self.forms = dict(formulation.forms)
        if forms_override:
            self.forms.update(forms_override)
        self.penalty_scale = penalty_scale
        self.forcing = forcing
        self.types = mesh.elem_types
        self.ops = {t: build_operators(t, N, formulation.kind) for t in self.types}
        self.n_elems = {t: len(mesh.blocks[t]) for t in self.types}
        self.dof_base, off = {}, 0
        for t in self.types:
            self.dof_base[t] = off
            off += self.n_elems[t] * FIELDS * self.ops[t].Np
        self.n_dof = off
        self.dtype = dtype
        self.device = torch.device(device) if device is not None else _default_device()
        self._dev = None
        self._data = None
        self._ref = None
        self._cub = {}

    # ------------------------------------------------------------ device side

    @property
    def device_mesh(self):
        if self._dev is None:
            if self.device is None or self.device.type != "cuda":
                raise RuntimeError("the hybridwave_b200 hot path needs a CUDA device")
            from .device import DeviceMesh
            self._dev = DeviceMesh(self, self.device, self.dtype)
        return self._dev

    def to_device(self, state):
        """dict of numpy/torch (K,4,Np) -> dict of contiguous device tensors."""
        out = {}
        for t in self.types:
            a = state[t]
            if isinstance(a, torch.Tensor):
                a = a.to(device=self.device, dtype=self.dtype)
            else:
                a = torch.as_tensor(np.asarray(a), dtype=self.dtype).to(self.device)
            out[t] = a.contiguous()
        return out

    def empty_state(self):
        return {t: torch.empty((self.n_elems[t], FIELDS, self.ops[t].Np), dtype=self.dtype,
                               device=self.device) for t in self.types}

    def zeros_state(self):
        return {t: torch.zeros((self.n_elems[t], FIELDS, self.ops[t].Np), dtype=self.dtype,
                               device=self.device) for t in self.types}

    def slots(self, state):
        """4-slot list (hex, wedge, pyramid, tet) of tensors / None."""
        s = [None] * 4
        if state is not None:
            for t in self.types:
                s[TYPE_ID[t]] = state[t]
        return s

    def stream_ptr(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def energy_device(self, q):
        """Discrete energy of a device state (hw_energy): a 0-d fp64 CUDA
        tensor (no host sync).  Same value as discrete_energy(state, disc)."""
        out = torch.empty(4, dtype=torch.float64, device=self.device)
        nat.check(nat.lib().hw_energy(self.device_mesh.struct, nat.fields(self.slots(q)),
                                      out.data_ptr(), self.stream_ptr()))
        return out.sum()

    def rhs_device(self, q, out=None, subset=None):
        """Device RHS: q, out dicts of CUDA tensors (no host copies)."""
        dm = self.device_mesh
        self.clear_forcing()          # compute_rhs adds the forcing itself
        dm.set_traces(0, None)        # hw_rhs fills trace set 0 with q's traces
        if dm.corr:                   # the corrections read the traces of q
            dm.compute_traces(nat.fields(self.slots(q)), 0, self.stream_ptr())
            self.apply_corrections()
        out = out if out is not None else self.empty_state()
        sub = nat.subset(subset) if subset is not None else None
        nat.check(nat.lib().hw_rhs(dm.struct, nat.fields(self.slots(q)),
                                   nat.fields(self.slots(out)), sub, self.stream_ptr()))
        self.clear_forcing()
        return out

    # ------------------------------------------------------------ public API

    def compute_rhs(self, state, time=0.0):
        """d(state)/dtau = diag(kappa, 1/rho) M^-1 (A state + forcing)
        (hybridwave/dg.py:492-506)."""
        on_host = not isinstance(next(iter(state.values())), torch.Tensor)
        q = self.to_device(state)
        out = self.rhs_device(q)
        if self.forcing is not None:
            self._add_forcing(out, time)
        if on_host:
            return {t: v.cpu().numpy() for t, v in out.items()}
        return out

    def _const(self, key, make):
        """Device copy of a host-side reference-layout array, built once."""
        if not hasattr(self, "_consts"):
            self._consts = {}
        if key not in self._consts:
            self._consts[key] = torch.as_tensor(np.ascontiguousarray(make()),
                                                dtype=torch.float64, device=self.device)
        return self._consts[key]

    def _mass_diag(self, t):
        """Per-node mass weights (hex w3 J, pyramid J; tet: J per element)."""
        d = self.data[t]
        if t == "hex":
            return self._const(("M", t), lambda: d.w3[None, :] * d.J)
        if t == "tet":
            return self._const(("M", t), lambda: d.J[:, 0])
        return self._const(("M", t), lambda: d.J)

    def apply_A(self, state):
        """R = A U: volume + surface residual, no mass inverse, no materials
        (hybridwave/dg.py:469-477).  On the device: the fused RHS kernels,
        then M diag(1/kappa, rho) applied to their output.  Host arrays in ->
        host arrays out (through HBM, like compute_rhs)."""
        on_host = not isinstance(next(iter(state.values())), torch.Tensor)
        rhs = self.rhs_device(self.to_device(state))
        out = {}
        for t in self.types:
            mat = self._const(("mat", t), lambda t=t: self.mesh.materials[t])
            r = rhs[t].double()
            r[:, 0] /= mat[:, 1][:, None]
            r[:, 1:] *= mat[:, 0][:, None, None]
            out[t] = self._apply_mass(t, r)
        if on_host:
            return {t: v.cpu().numpy() for t, v in out.items()}
        return out

    def _apply_mass(self, t, v):
        if t == "wedge":                   # LSC-DG: identity mass (dg.py:486-487)
            return v
        m = self._mass_diag(t)
        if t == "tet":
            Mref = self._const(("Mref", t), lambda: self.ops[t].M_ref)
            return (v @ Mref.T) * m[:, None, None]
        return v * m[:, None, :]

    def apply_mass_inverse(self, t, residual_t):
        """hybridwave/dg.py:479-490 on the device: hex / (w3 J), tet
        invM_ref / J, wedge identity, pyramid / J.  A CUDA tensor stays on
        the device; a host array is copied in and the result copied back."""
        on_host = not isinstance(residual_t, torch.Tensor)
        r = torch.as_tensor(np.asarray(residual_t) if on_host else residual_t,
                            dtype=torch.float64).to(self.device)
        if t == "wedge":
            out = r.clone()
        elif t == "tet":
            Minv = self._const(("Minv", t), lambda: self.ops[t].invM_ref)
            out = (r @ Minv.T) / self._mass_diag(t)[:, None, None]
        else:
            out = r / self._mass_diag(t)[:, None, :]
        return out.cpu().numpy() if on_host else out

    def compute_traces(self, state):
        """Own-side traces at the reference's stored face points in its flat
        layout, (4, trace_size) (hybridwave/dg.py:299-316), on the device:
        state @ Vf^T per type, wedge traces x 1/sqrt(J).  Diagnostic: the
        stage kernels never form this buffer (they read neighbour state or
        the compact published traces)."""
        on_host = not isinstance(next(iter(state.values())), torch.Tensor)
        q = self.to_device(state)
        out = torch.empty((FIELDS, self.trace_size), dtype=torch.float64, device=self.device)
        for t in self.types:
            op = self.ops[t]
            Vf = self._const(("Vf", t), lambda op=op: op.Vf)
            tr = q[t].double() @ Vf.T                               # (K, 4, Nfp)
            if t == "wedge":
                tr = tr * self._const(("isJf", t),
                                      lambda: self.data["wedge"].invsqrtJ_face)[:, None, :]
            b = self.trace_bases[t]
            n = self.n_elems[t] * op.face_offsets[-1]
            out[:, b:b + n] = tr.transpose(0, 1).reshape(FIELDS, n)
        return out.cpu().numpy() if on_host else out

    def apply_mass(self, t, v):
        """Host M v (diagnostics / tests)."""
        d = self.data[t]
        if t == "hex":
            return v * (d.w3[None, None, :] * d.J[:, None, :])
        if t == "tet":
            return (v @ self.ops[t].M_ref.T) * d.J[:, 0][:, None, None]
        if t == "wedge":
            return v.copy()
        return v * d.J[:, None, :]

    # ------------------------------------------------------------ forcing / projection

    def _basis_values(self, t, abc):
        op = self.ops[t]
        if t == "hex":
            return bas.hex_nodal_eval(self.N, "GL" if self.formulation.kind == "GL" else "SEM",
                                      duffy_map("hex", abc)).V
        if t == "tet":
            return bas.tet_orthobasis_eval(self.N, abc).V @ op.Vinv
        if t == "wedge":
            return bas.wedge_orthobasis_eval(self.N, abc).V
        return bas.pyramid_seminodal_eval(self.N, abc).V

    def _cubature(self, t, which):
        """Cubature data for projection ('cub', degree N) and error norms
        ('over', degree N+2), dg.py:177-188."""
        key = (t, which)
        if key not in self._cub:
            rule = element_rule(t, self.N if which == "cub" else self.N + 2)
            verts = self.mesh.element_vertices(t)
            x = map_points(t, verts, rule.collapsed)
            J = jacobian_det_fast(t, verts, rule.collapsed)
            self._cub[key] = (rule.weights, self._basis_values(t, rule.collapsed), x, J)
        return self._cub[key]

    def _forcing_ops(self, t):
        """Device operands of hw_forcing for type t, built once: B = [invM_ref]
        V^T diag(w) (Np, nq), scale = J (sqrt(J) wedge) at the cubature
        points (K, nq), the per-node mass inverse (K, Np), and the cubature
        points themselves for device-evaluated forcing (hybridwave/dg.py:
        177-188, 479-490, 508-515)."""
        cache = self.__dict__.setdefault("_frc_ops", {})
        if t not in cache:
            w, V, x, J = self._cubature(t, "cub")
            B = V.T * w[None, :]
            if t == "tet":
                B = self.ops[t].invM_ref @ B
            scale = np.sqrt(J) if t == "wedge" else J
            d, Np = self.data[t], self.ops[t].Np
            if t == "hex":
                nodefac = 1.0 / (d.w3[None, :] * d.J)
            elif t == "tet":
                nodefac = np.repeat(1.0 / d.J[:, :1], Np, axis=1)
            elif t == "wedge":
                nodefac = np.ones((self.n_elems[t], Np))
            else:
                nodefac = 1.0 / d.J
            dev = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64,
                                            device=self.device)
            cache[t] = {"B": dev(B), "scale": dev(scale), "nodefac": dev(nodefac),
                        "x": x, "x_dev": None, "nq": int(B.shape[1])}
        return cache[t]

    def forcing_values(self, t, time):
        """The forcing callback at type t's cubature points as a (K, nq) fp64
        CUDA tensor.  A callback with ``on_device = True`` is called with the
        points as a CUDA tensor (no host work); otherwise with numpy points,
        as in the reference, and the values are copied to the device."""
        op = self._forcing_ops(t)
        if getattr(self.forcing, "on_device", False):
            if op["x_dev"] is None:
                op["x_dev"] = torch.as_tensor(op["x"], dtype=torch.float64, device=self.device)
            f = self.forcing(op["x_dev"], time)
            return torch.as_tensor(f, dtype=torch.float64, device=self.device).contiguous()
        f = np.ascontiguousarray(np.asarray(self.forcing(op["x"], time), dtype=np.float64))
        return torch.as_tensor(f).to(self.device, non_blocking=False)

    def forcing_buffer(self):
        if getattr(self, "_frc_buf", None) is None:
            self._frc_buf = self.zeros_state()
        return self._frc_buf

    def set_forcing(self, time):
        """Fill the forcing buffer with kappa M^-1 (forcing integral) at `time`
        (hw_forcing) and point the mesh's frc slots at it: the next
        hw_rhs / hw_lsrk_stage / hw_ab_step add it to dp/dtau in their
        epilogues.  Returns the buffer dict."""
        dm, L, st = self.device_mesh, nat.lib(), self.stream_ptr()
        buf = self.forcing_buffer()
        keep = []
        for t in self.types:
            op = self._forcing_ops(t)
            f = self.forcing_values(t, time)
            keep.append(f)
            nat.check(L.hw_forcing(dm.struct, TYPE_ID[t], f.data_ptr(), op["B"].data_ptr(),
                                   op["scale"].data_ptr(), op["nodefac"].data_ptr(), op["nq"],
                                   1.0, buf[t].data_ptr(), 0.0, None, 1, st))
            dm.struct.frc[TYPE_ID[t]] = buf[t].data_ptr()
        self._frc_keep = keep           # alive until the kernels ran
        return buf

    def clear_forcing(self):
        if self._dev is not None:
            for i in range(4):
                self._dev.struct.frc[i] = None

    @property
    def has_corrections(self):
        return bool(self.device_mesh.corr)

    def apply_corrections(self, after_forcing=False, rows=None, zero=True):
        """Extra-RHS rows of the tets / pyramids across non-affine wedge triangles: the
        reference's face-cubature integral minus the kernels' nodal lift
        (hw_wedge_face_correction) from the current input traces
        (mesh->tr_in), installed in the mesh's frc slots (accumulates onto a
        forcing term set just before).  rows: a subset of the correction
        rows (partitioned runs apply the rows of ghost wedges after the halo
        exchange); zero=False adds onto the rows already accumulated."""
        dm, L, st = self.device_mesh, nat.lib(), self.stream_ptr()
        if not dm.corr:
            return
        buf = self.forcing_buffer()
        if zero and not after_forcing:       # rows hold the last stage's values
            for t, c in dm.corr.items():
                buf[t].index_fill_(0, c["elems"], 0.0)
        for t, c in (dm.corr if rows is None else rows).items():
            nat.check(L.hw_wedge_face_correction(dm.struct, TYPE_ID[t], c["n"],
                                                 c["idata"].data_ptr(), c["fdata"].data_ptr(),
                                                 c["L"].data_ptr(), c["P"].data_ptr(), c["nq"],
                                                 c["nfn"], buf[t].data_ptr(), st))
        for t in dm.corr:
            dm.struct.frc[TYPE_ID[t]] = buf[t].data_ptr()

    def prepare_stage(self, time):
        """Extra RHS of the next fused stage: forcing at `time` (if any), then
        the face corrections.  Call after the stage's input traces are set.
        Returns True when the mesh's frc slots were installed."""
        on = False
        self.clear_forcing()
        if self.forcing is not None:
            self.set_forcing(time)
            on = True
        if self._dev is not None and self._dev.corr:
            self.apply_corrections(after_forcing=self.forcing is not None)
            on = True
        return on

    def _add_forcing(self, out, time):
        """out (device dict) += the forcing term at `time`, on the device."""
        dm, L, st = self.device_mesh, nat.lib(), self.stream_ptr()
        for t in self.types:
            op = self._forcing_ops(t)
            f = self.forcing_values(t, time)
            nat.check(L.hw_forcing(dm.struct, TYPE_ID[t], f.data_ptr(), op["B"].data_ptr(),
                                   op["scale"].data_ptr(), op["nodefac"].data_ptr(), op["nq"],
                                   1.0, out[t].data_ptr(), 0.0, None, 0, st))

    def project(self, fields_fn, time=0.0):
        """L2 projection of callable fields (dg.py:521-548); host numpy."""
        state = {}
        for t in self.types:
            if t == "hex":
                n1 = self.ops["hex"].nodes1d
                i, j, k = np.meshgrid(n1, n1, n1, indexing="ij")
                pts = np.column_stack([i.ravel(), j.ravel(), k.ravel()])
                x = map_points("hex", self.mesh.element_vertices("hex"), pts)
                state[t] = np.moveaxis(np.asarray(fields_fn(x, time)), -1, 1)
                continue
            w, V, x, J = self._cubature(t, "cub")
            vals = np.moveaxis(np.asarray(fields_fn(x, time)), -1, 1)
            if t == "tet":
                state[t] = ((vals * w[None, None, :]) @ V) @ self.ops[t].invM_ref
            elif t == "wedge":
                state[t] = (vals * (w[None, :] * np.sqrt(J))[:, None, :]) @ V
            else:
                raw = (vals * (w[None, :] * J)[:, None, :]) @ V
                Jr = jacobian_det_fast(t, self.mesh.element_vertices(t), self.ops[t].level_abc)
                state[t] = raw / Jr[:, None, :]
        return state

    def eval_at(self, t, state_t, which="over"):
        w, V, x, J = self._cubature(t, which)
        vals = _host(state_t) @ V.T
        if t == "wedge":
            vals = vals / np.sqrt(J)[:, None, :]
        return vals

    def l2_error(self, state, exact_fn, time=0.0):
        """Over-integrated L2 errors {p, u, total} (hybridwave/dg.py:558-572),
        on the device: the state is evaluated at the degree-(N+2) cubature
        points by a matmul with the stored basis values, the exact solution
        is evaluated there (on the device when ``exact_fn.on_device``), and
        the weighted squares are reduced with one host read at the end.
        Host arrays or CUDA tensors in."""
        dev = self.device
        num_p = torch.zeros((), dtype=torch.float64, device=dev)
        num_u = torch.zeros((), dtype=torch.float64, device=dev)
        for t in self.types:
            w, V, x, J = self._cubature(t, "over")
            c = self.__dict__.setdefault("_l2_ops", {})
            if t not in c:
                Vd = torch.as_tensor(V, dtype=torch.float64, device=dev)
                wJ = torch.as_tensor(w[None, :] * J, dtype=torch.float64, device=dev)
                isj = (torch.as_tensor(1.0 / np.sqrt(J), dtype=torch.float64, device=dev)
                       if t == "wedge" else None)
                c[t] = (Vd, wJ, isj)
            Vd, wJ, isj = c[t]
            s_ = state[t]
            s_ = (s_ if isinstance(s_, torch.Tensor)
                  else torch.as_tensor(np.asarray(s_))).to(dev, torch.float64)
            vals = s_ @ Vd.T                                     # (K, 4, nq)
            if isj is not None:
                vals = vals * isj[:, None, :]
            if getattr(exact_fn, "on_device", False):
                ex = exact_fn(torch.as_tensor(x, dtype=torch.float64, device=dev), time)
            else:
                ex = torch.as_tensor(np.asarray(exact_fn(x, time)), dtype=torch.float64)
            ex = ex.to(dev).movedim(-1, 1)
            d2 = (vals - ex) ** 2
            num_p = num_p + (d2[:, 0] * wJ).sum()
            num_u = num_u + (d2[:, 1:] * wJ[:, None, :]).sum()
        p_, u_ = (float(v) for v in torch.stack([num_p, num_u]).cpu())
        return {"p": np.sqrt(p_), "u": np.sqrt(u_), "total": np.sqrt(p_ + u_)}

    def state_to_vector(self, state):
        return np.concatenate([_host(state[t]).ravel() for t in self.types])

    def vector_to_state(self, vec):
        out = {}
        for t in self.types:
            b = self.dof_base[t]
            n = self.n_elems[t] * FIELDS * self.ops[t].Np
            out[t] = vec[b:b + n].reshape(self.n_elems[t], FIELDS, self.ops[t].Np)
        return out

    # ------------------------------------------------------------ reference layout

    @property
    def data(self):
        self._ensure_reference_layout()
        return self._data

    @property
    def gather_idx(self):
        self._ensure_reference_layout()
        return self._ref["gather"]

    @property
    def bnd_mask(self):
        self._ensure_reference_layout()
        return self._ref["bnd"]

    @property
    def trace_size(self):
        return sum(self.n_elems[t] * self.ops[t].face_offsets[-1] for t in self.types)

    @property
    def trace_bases(self):
        b, off = {}, 0
        for t in self.types:
            b[t] = off
            off += self.n_elems[t] * self.ops[t].face_offsets[-1]
        return b

    def _ensure_reference_layout(self):
        if self._data is not None:
            return
        data = {}
        for t in self.types:
            data[t] = self._type_data(t)
        self._data = data
        self._ref = self._build_gather()

    def _type_data(self, t):
        """hybridwave/dg.py:139-192 (geometry at the reference's volume and
        stored face points)."""
        op = self.ops[t]
        d = _TypeData()
        verts = self.mesh.element_vertices(t)
        d.verts = verts
        d.diam = np.linalg.norm(verts.max(axis=1) - verts.min(axis=1), axis=1)
        if t == "hex":
            n1 = op.nodes1d
            i, j, k = np.meshgrid(n1, n1, n1, indexing="ij")
            pts = np.column_stack([i.ravel(), j.ravel(), k.ravel()])
        elif t == "tet":
            pts = np.array([[-0.5, -0.5, -0.5]])
        elif t == "wedge":
            pts = op.cub.collapsed
        else:
            pts = op.level_abc
        x, J, G, gradJ = geometric_factors_batch(t, verts, pts, label=t)
        d.J, d.G = J, G
        if t == "wedge":
            d.gJfac = -gradJ / (2.0 * J[..., None])
        if t == "pyramid":
            d.J_row = J
        if t == "hex":
            d.x_nodes = x
            d.w3 = np.einsum("i,j,k->ijk", op.weights1d, op.weights1d, op.weights1d).ravel()
        K = len(verts)
        tot = op.face_offsets[-1]
        d.wJs = np.empty((K, tot))
        d.normals = np.empty((K, tot, 3))
        d.x_face = np.empty((K, tot, 3))
        for f, (p2, w2) in enumerate(zip(op.face_pts2d, op.face_wts)):
            sl = slice(op.face_offsets[f], op.face_offsets[f + 1])
            xf, Js, nrm = face_geometry_batch(t, verts, f, p2)
            d.x_face[:, sl] = xf
            d.wJs[:, sl] = w2[None, :] * Js
            d.normals[:, sl] = nrm
        if t == "wedge":
            abc_f = inverse_duffy_map("wedge", op.face_rst)
            _, Jf, _, _ = geometric_factors_batch("wedge", verts, abc_f, label=t)
            d.invsqrtJ_face = 1.0 / np.sqrt(Jf)
        mat = self.mesh.materials[t]
        d.rhoc = mat[:, 0] * np.sqrt(mat[:, 1] / mat[:, 0])
        return d

    def _build_gather(self):
        """Global face-point gather (dg.py:217-285) from the connectivity
        orientation codes and the stored rules' symmetry permutations,
        verified geometrically."""
        bases = self.trace_bases
        size = self.trace_size
        gather = np.arange(size)
        bnd = np.zeros(size, dtype=bool)
        tau_p = np.empty(size)
        tau_u = np.empty(size)
        perms = {}
        for t in self.types:
            op = self.ops[t]
            for f, (ftype, _) in enumerate(FACES[t]):
                if ftype not in perms:
                    perms[ftype] = face_symmetry_perms(ftype, op.face_pts2d[f])
        for t in self.types:
            op, d = self.ops[t], self.data[t]
            tot = op.face_offsets[-1]
            nbr, code = self.mesh.nbr[t], self.mesh.face_code[t]
            K = self.n_elems[t]
            for f, (ftype, _) in enumerate(FACES[t]):
                off, nq = op.face_offsets[f], op.face_offsets[f + 1] - op.face_offsets[f]
                me = bases[t] + np.arange(K)[:, None] * tot + off + np.arange(nq)[None, :]
                isb = nbr[:, f, 0] < 0
                bnd[me[isb].ravel()] = True
                zm = d.rhoc
                zp = d.rhoc.copy()
                for t2 in self.types:
                    sel = (~isb) & (nbr[:, f, 0] == TYPE_ID[t2])
                    if not sel.any():
                        continue
                    op2 = self.ops[t2]
                    k2, f2 = nbr[sel, f, 1], nbr[sel, f, 2]
                    tot2 = op2.face_offsets[-1]
                    p = perms[ftype][code[sel, f]]                     # (n, nq)
                    src = bases[t2] + k2[:, None] * tot2 + op2.face_offsets[f2][:, None] + p
                    gather[me[sel].ravel()] = src.ravel()
                    zp[sel] = self.data[t2].rhoc[k2]
                    # geometric verification of the coincidence
                    xs = self.data[t2].x_face[k2[:, None], op2.face_offsets[f2][:, None] + p]
                    err = np.linalg.norm(xs - d.x_face[sel][:, off:off + nq], axis=2).max(axis=1)
                    tol = 1e-10 * np.maximum(d.diam[sel], self.data[t2].diam[k2])
                    if np.any(err > tol):
                        raise ValueError(f"face cubature points do not coincide on {t} face {f}")
                avg = 0.5 * (zm + zp)
                tau_p[me] = (1.0 / avg)[:, None]
                tau_u[me] = avg[:, None]
        for t in self.types:
            d = self.data[t]
            tot = self.ops[t].face_offsets[-1]
            sl = slice(bases[t], bases[t] + self.n_elems[t] * tot)
            d.tau_p = tau_p[sl].reshape(self.n_elems[t], tot)
            d.tau_u = tau_u[sl].reshape(self.n_elems[t], tot)
        return {"gather": gather, "bnd": bnd}


def _host(a):
    if isinstance(a, torch.Tensor):
        return a.detach().cpu().numpy()
    return np.asarray(a)


def discrete_energy(state, disc):
    """U^T M U with material weights (hybridwave/dg.py:655-674)."""
    total = 0.0
    for t in disc.types:
        s = _host(state[t])
        d = disc.data[t]
        mat = disc.mesh.materials[t]
        if t == "hex":
            en = (d.w3[None, None, :] * d.J[:, None, :] * s ** 2).sum(axis=2)
        elif t == "tet":
            en = np.einsum("kfi,ij,kfj->kf", s, disc.ops[t].M_ref, s) * d.J[:, 0][:, None]
        elif t == "wedge":
            en = (s ** 2).sum(axis=2)
        else:
            en = (d.J[:, None, :] * s ** 2).sum(axis=2)
        total += float(np.sum(en[:, 0] / mat[:, 1]))
        total += float(np.sum(en[:, 1:] * mat[:, 0][:, None]))
    return total
