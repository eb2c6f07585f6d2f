"""Python mirror of the reference's geoshoot API over the C ABI.

Same names, argument meaning and error behaviour as the reference's C++ API
(/root/reference/proj/include/geoshoot/{core,kernel_exact,octree,bh_kernel,
shooting}.hpp), so the parity tests read like the reference's own tests:

  reference (C++)                          here
  ---------------------------------------  -------------------------------------
  hamiltonian(q, p, sigma)                 Geoshoot.hamiltonian(q, p, sigma)
  hamiltonian_gradients(q, p, sigma)       Geoshoot.hamiltonian_gradients(...)
  exact_velocity(x, q, p, sigma)           Geoshoot.exact_velocity(...)
  hessian_products(q, p, a, b, sigma)      Geoshoot.hessian_products(...)
  Octree::build(q, p)                      Geoshoot.build_tree(q, p) -> Octree
  bh_velocity / bh_hamiltonian_gradients   Octree.bh_velocity / .bh_hamiltonian_gradients
  shoot_forward / objective / evaluate     Geoshoot.shoot_forward / .objective / .evaluate
  backward_gradient / warp_points          Geoshoot.backward_gradient / .warp_points

Arrays are numpy float64 (n, 3) -- the reference's std::vector<Vec3> layout.
Exceptions mirror core.hpp:69-116.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


# ---- exceptions (core.hpp:69-116) -------------------------------------------
class GeoshootError(RuntimeError):
    pass


class DimensionMismatch(ValueError):
    pass


class OutOfBounds(ValueError):
    pass


class EmptyTree(GeoshootError):
    pass


class NonFiniteState(GeoshootError):
    def __init__(self, timestep: int):
        super().__init__(f"non-finite state at timestep {timestep}")
        self.timestep = timestep


class ConfigMismatch(ValueError):
    pass


class ConfigError(ValueError):
    VIOLATIONS = ("NonPositiveSigma", "NonPositiveLambda", "ZeroTimesteps", "NonPositiveThreshold")

    def __init__(self, mask: int):
        self.violations = [v for k, v in enumerate(self.VIOLATIONS) if mask & (1 << k)]
        super().__init__("invalid shooting config: " + " ".join(self.violations))


class DeviceError(GeoshootError):
    pass


class ParseError(GeoshootError):
    def __init__(self, line: int, msg: str):
        super().__init__(msg)
        self.line = line


class UnsupportedFormat(GeoshootError):
    pass


class DegenerateConfiguration(GeoshootError):
    pass


# ---- point-cloud files (pipeline.hpp:52-68; host-side, no device needed) -----
XYZ, VTK = 0, 1


def format_for_path(path: str) -> int:
    return L.load().gs_format_for_path(path.encode())


def _io_check(lib, st):
    if st == L.GS_OK:
        return
    msg = (lib.gs_last_io_error() or b"").decode()
    if st == L.GS_PARSE_ERROR:
        raise ParseError(lib.gs_last_parse_line(), msg)
    if st == L.GS_UNSUPPORTED_FORMAT:
        raise UnsupportedFormat(msg)
    if st == L.GS_INVALID_ARGUMENT:
        raise ValueError(msg)
    raise OSError(msg)


def read_points(path: str, fmt: int = None) -> np.ndarray:
    lib = L.load()
    fmt = format_for_path(path) if fmt is None else fmt
    n = C.c_int64()
    _io_check(lib, lib.gs_read_points(path.encode(), fmt, None, 0, C.byref(n)))
    out = np.empty((n.value, 3))
    _io_check(lib, lib.gs_read_points(path.encode(), fmt, _p(out), n.value, C.byref(n)))
    return out


def write_points(points, path: str, fmt: int = None, header=()):
    lib = L.load()
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    fmt = format_for_path(path) if fmt is None else fmt
    hdr = (C.c_char_p * max(1, len(header)))(*[h.encode() for h in header])
    _io_check(lib, lib.gs_write_points(path.encode(), fmt, len(pts), _p(pts), hdr, len(header)))


# ---- config (core.hpp:184-213) ------------------------------------------------
EXACT, BARNES_HUT = L.GS_EXACT, L.GS_BARNES_HUT
EULER, RK4 = L.GS_EULER, L.GS_RK4
F64, F32 = L.GS_F64, L.GS_F32


@dataclass
class ShootingConfig:
    sigma: float = 2.0
    lambda_: float = 1.0
    timesteps: int = 40
    backend: int = EXACT
    threshold_multiplier: float = 3.0
    integrator: int = EULER
    precision: int = F64
    literal_mean_dot: bool = False  # GEOSHOOT_BH_LITERAL_MEAN_DOT (bh_kernel.cpp:19-26)
    exact_cutoff: bool = False  # FP32 exact flows: skip tile pairs whose weights underflow to 0
    flags: int = 0              # raw gs_config.flags bits (GS_FLAG_*)

    def opening_threshold(self) -> float:
        return self.threshold_multiplier * self.sigma

    def c(self) -> L.gs_config:
        return L.gs_config(self.sigma, self.lambda_, self.timesteps, self.backend,
                           self.threshold_multiplier, self.integrator, self.precision,
                           1 if self.literal_mean_dot else 0,
                           self.flags | (L.GS_FLAG_EXACT_CUTOFF if self.exact_cutoff else 0))


def _arr(a, name="array") -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[1] != 3:
        raise ValueError(f"{name}: expected shape (n, 3), got {a.shape}")
    return a


def _p(a):
    return None if a is None else a.ctypes.data_as(L._d)


def _require_aligned(n1, n2, where):
    if n1 != n2:  # require_aligned, core.hpp:172-178
        raise DimensionMismatch(f"{where}: point/momentum counts differ ({n1} vs {n2})")


@dataclass
class Trajectory:
    """GeodesicTrajectory (core.hpp:262-274): states[k] = (q_k, p_k), k = 0..T."""
    q: np.ndarray  # (T+1, n, 3)
    p: np.ndarray

    @property
    def states(self):
        return list(zip(self.q, self.p))

    def timesteps(self):
        return self.q.shape[0] - 1

    def final_state(self):
        return self.q[-1], self.p[-1]


@dataclass
class Evaluation:
    report: dict
    gradient: np.ndarray
    stats: dict = field(default_factory=dict)


class Geoshoot:
    """A device context (gs_ctx): a CUDA stream + workspaces on one B200, or --
    with ``devices=[...]`` -- a multi-device context (gs_create_multi) whose
    shooting calls (shoot_forward, objective, evaluate, optimize, flows) shard
    the target points across the devices, the per-stage exchange fused into
    the stage epilogues as peer stores."""

    def __init__(self, device: int = 0, devices=None):
        self.lib = L.load()
        st = C.c_int(0)
        if devices is None:
            self.ctx = self.lib.gs_create(device, C.byref(st))
        else:
            arr = (C.c_int32 * len(devices))(*devices)
            self.ctx = self.lib.gs_create_multi(len(devices), arr, C.byref(st))
        if not self.ctx:
            raise DeviceError(f"gs_create failed ({st.value}): {self._err()}")

    @property
    def device_count(self) -> int:
        return self.lib.gs_ctx_device_count(self.ctx)

    @property
    def peer_stores(self) -> bool:
        return bool(self.lib.gs_ctx_peer_stores(self.ctx))

    PHASES = ("kernel", "build", "bbox_keys", "sort", "topology", "aggregate", "adjoint_kernel")

    def profile(self, enable: bool = True):
        """Event timing of the dominant kernels inside shooting calls (gs_profile)."""
        self.check(self.lib.gs_profile(self.ctx, 1 if enable else 0))

    def profile_phases(self) -> dict:
        k = len(self.PHASES)
        ms = np.zeros(k)
        cnt = (C.c_int64 * k)()
        self.check(self.lib.gs_profile_phases(self.ctx, _p(ms), cnt, k))
        return {name: {"ms": float(ms[i]), "count": int(cnt[i])} for i, name in enumerate(self.PHASES)}

    def trace(self, enable: bool = True):
        """Kernel start-time trace (gs_trace): valid inside captured graphs."""
        self.check(self.lib.gs_trace(self.ctx, 1 if enable else 0))

    def trace_read(self, max_entries: int = 16384):
        """[(unit, line, t_ns)] of the traced kernel starts since the last read."""
        tags = np.zeros(max_entries, np.uint64)
        times = np.zeros(max_entries, np.uint64)
        cnt = C.c_int64()
        self.check(self.lib.gs_trace_read(self.ctx, tags.ctypes.data_as(C.POINTER(C.c_uint64)),
                                          times.ctypes.data_as(C.POINTER(C.c_uint64)), max_entries,
                                          C.byref(cnt)))
        k = cnt.value
        return [(int(t) >> 16, int(t) & 0xffff, int(v)) for t, v in zip(tags[:k], times[:k])]

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.gs_destroy(self.ctx)
            self.ctx = None

    __del__ = close

    def _err(self) -> str:
        m = self.lib.gs_last_error(getattr(self, "ctx", None))
        return m.decode() if m else ""

    def check(self, st: int):
        if st == L.GS_OK:
            return
        msg = self._err()
        if st == L.GS_NONFINITE:
            raise NonFiniteState(self.lib.gs_last_nonfinite_step(self.ctx))
        if st == L.GS_CONFIG_ERROR:
            raise ConfigError(self.lib.gs_last_config_violations(self.ctx))
        if st == L.GS_DIMENSION_MISMATCH:
            raise DimensionMismatch(msg)
        if st == L.GS_CONFIG_MISMATCH:
            raise ConfigMismatch(msg)
        if st == L.GS_EMPTY_TREE:
            raise EmptyTree(msg)
        if st == L.GS_OUT_OF_BOUNDS:
            raise OutOfBounds(msg)
        if st == L.GS_INVALID_ARGUMENT:
            raise ValueError(msg)
        if st == L.GS_DEGENERATE:
            raise DegenerateConfiguration(msg)
        raise DeviceError(f"status {st}: {msg}")

    # ---- kernel_exact -----------------------------------------------------
    def hamiltonian(self, q, p, sigma, precision=F64) -> float:
        q, p = _arr(q, "q"), _arr(p, "p")
        _require_aligned(len(q), len(p), "hamiltonian")
        h = C.c_double()
        self.check(self.lib.gs_hamiltonian(self.ctx, precision, len(q), _p(q), _p(p), sigma,
                                           C.byref(h)))
        return h.value

    def hamiltonian_with_gradients(self, q, p, sigma, precision=F64):
        q, p = _arr(q, "q"), _arr(p, "p")
        _require_aligned(len(q), len(p), "hamiltonian_gradients")
        dp, dq = np.empty_like(q), np.empty_like(q)
        h = C.c_double()
        self.check(self.lib.gs_exact_rhs(self.ctx, precision, len(q), _p(q), _p(p), sigma, _p(dp),
                                         _p(dq), C.byref(h)))
        return h.value, dp, dq

    def hamiltonian_gradients(self, q, p, sigma, precision=F64):
        _, dp, dq = self.hamiltonian_with_gradients(q, p, sigma, precision)
        return dp, dq

    def exact_velocity(self, x, q, p, sigma, precision=F64):
        x, q, p = _arr(x, "x"), _arr(q, "q"), _arr(p, "p")
        _require_aligned(len(q), len(p), "exact_velocity")
        v = np.empty_like(x)
        self.check(self.lib.gs_exact_velocity(self.ctx, precision, len(x), _p(x), len(q), _p(q),
                                              _p(p), sigma, _p(v)))
        return v

    def hessian_products(self, q, p, alpha, beta, sigma, precision=F64):
        q, p, a, b = _arr(q), _arr(p), _arr(alpha), _arr(beta)
        _require_aligned(len(q), len(p), "hessian_products")
        _require_aligned(len(q), len(a), "hessian_products(alpha)")
        _require_aligned(len(q), len(b), "hessian_products(beta)")
        out = [np.empty_like(q) for _ in range(4)]
        self.check(self.lib.gs_hessian_products(self.ctx, precision, len(q), _p(q), _p(p), _p(a),
                                                _p(b), sigma, *map(_p, out)))
        return tuple(out)  # pq_alpha, pp_alpha, qq_beta, qp_beta

    # ---- octree -------------------------------------------------------------
    def set_bh_walk(self, kernel: int = -1, windows: int = -1):
        """Process-wide Barnes-Hut walk override (gs_set_bh_walk): kernel 0 by regime,
        1 independent walks, 3 group walk, 4 split; windows 0 auto or K; -1 = default."""
        st = self.lib.gs_set_bh_walk(int(kernel), int(windows))
        if st:
            raise ValueError(f"gs_set_bh_walk({kernel}, {windows}): invalid choice")

    def set_exact_pairs(self, mode: int = -1):
        """Process-wide exact FP32 all-pairs formulation (gs_set_exact_pairs): 0 by size,
        1 gather (ordered pairs per target), 2 symmetric (unordered pairs once); -1 default."""
        st = self.lib.gs_set_exact_pairs(int(mode))
        if st:
            raise ValueError(f"gs_set_exact_pairs({mode}): invalid choice")

    def exact_pairs_plan(self, n: int, precision=F32) -> int:
        """Tiles T of the symmetric exact RHS an unsharded n-point problem takes now
        (0: the gather kernel) -- gs_exact_pairs_plan."""
        t = C.c_int32()
        self.check(self.lib.gs_exact_pairs_plan(int(precision), int(n), C.byref(t)))
        return t.value

    def set_literal_mean_dot(self, enable: bool):
        """Tree-level BH calls on this context use the reference's
        GEOSHOOT_BH_LITERAL_MEAN_DOT aggregate dot scale 1/count (bh_kernel.cpp:19-26)."""
        self.check(self.lib.gs_set_literal_mean_dot(self.ctx, 1 if enable else 0))

    def build_tree(self, q, p, precision=F64) -> "Octree":
        q, p = _arr(q, "q"), _arr(p, "p")
        _require_aligned(len(q), len(p), "Octree::build")
        h = C.c_void_p()
        self.check(self.lib.gs_tree_build(self.ctx, precision, len(q), _p(q), _p(p), C.byref(h)))
        return Octree(self, h, q, p)

    # ---- shooting -----------------------------------------------------------
    def shoot_forward(self, q0, p0, cfg: ShootingConfig, keep_trajectory=True):
        q0, p0 = _arr(q0, "q0"), _arr(p0, "p0")
        _require_aligned(len(q0), len(p0), "shoot_forward")
        n, T = len(q0), cfg.timesteps
        c = cfg.c()
        st = L.gs_stats()
        e = C.c_double()
        if keep_trajectory:
            tq = np.empty((T + 1, n, 3)) if T >= 0 else None
            tp = np.empty((T + 1, n, 3)) if T >= 0 else None
            self.check(self.lib.gs_shoot_forward(self.ctx, C.byref(c), n, _p(q0), _p(p0), _p(tq),
                                                 _p(tp), None, None, C.byref(e), C.byref(st)))
            return Trajectory(tq, tp)
        fq, fp = np.empty_like(q0), np.empty_like(q0)
        self.check(self.lib.gs_shoot_forward(self.ctx, C.byref(c), n, _p(q0), _p(p0), None, None,
                                             _p(fq), _p(fp), C.byref(e), C.byref(st)))
        return fq, fp, e.value, st.as_dict()

    def objective(self, q0, p0, target, cfg: ShootingConfig) -> dict:
        q0, p0, t = _arr(q0), _arr(p0), _arr(target)
        _require_aligned(len(q0), len(p0), "shoot_forward")
        _require_aligned(len(q0), len(t), "objective(target)")
        c = cfg.c()
        r = L.gs_report()
        self.check(self.lib.gs_objective(self.ctx, C.byref(c), len(q0), _p(q0), _p(p0), _p(t),
                                         C.byref(r)))
        return {"energy": r.energy, "attachment": r.attachment, "total": r.total,
                "residual_sse": r.residual_sse}

    def backward_gradient(self, traj: Trajectory, target, cfg: ShootingConfig):
        tq = np.ascontiguousarray(traj.q, dtype=np.float64)
        tp = np.ascontiguousarray(traj.p, dtype=np.float64)
        t = _arr(target)
        _require_aligned(tq.shape[1], len(t), "backward_gradient(target)")
        g = np.empty_like(t)
        c = cfg.c()
        self.check(self.lib.gs_backward_gradient(self.ctx, C.byref(c), tq.shape[1], tq.shape[0],
                                                 _p(tq), _p(tp), _p(t), _p(g)))
        return g

    def warp_points(self, traj: Trajectory, x, cfg: ShootingConfig):
        tq = np.ascontiguousarray(traj.q, dtype=np.float64)
        tp = np.ascontiguousarray(traj.p, dtype=np.float64)
        x = _arr(x, "x")
        y = np.empty_like(x)
        c = cfg.c()
        self.check(self.lib.gs_warp_points(self.ctx, C.byref(c), tq.shape[1], tq.shape[0], _p(tq),
                                           _p(tp), len(x), _p(x), _p(y)))
        return y

    def evaluate(self, q0, p0, target, cfg: ShootingConfig) -> Evaluation:
        q0, p0, t = _arr(q0), _arr(p0), _arr(target)
        _require_aligned(len(q0), len(p0), "shoot_forward")
        _require_aligned(len(q0), len(t), "objective(target)")
        c = cfg.c()
        r = L.gs_report()
        g = np.empty_like(q0)
        st = L.gs_stats()
        self.check(self.lib.gs_evaluate(self.ctx, C.byref(c), len(q0), _p(q0), _p(p0), _p(t),
                                        C.byref(r), _p(g), C.byref(st)))
        rep = {"energy": r.energy, "attachment": r.attachment, "total": r.total,
               "residual_sse": r.residual_sse}
        return Evaluation(rep, g, st.as_dict())

    def optimize(self, q0, target, cfg: ShootingConfig, max_iterations=200, memory=10,
                 gradient_tolerance=1e-6, relative_objective_tolerance=1e-9,
                 sufficient_decrease=1e-4, curvature=0.9, max_trials=20):
        """optimize() (optimizer.cpp:301-351): L-BFGS over p0 from 0."""
        q0, t = _arr(q0, "q0"), _arr(target, "target")
        _require_aligned(len(q0), len(t), "optimize")
        c = cfg.c()
        oc = L.gs_opt_config(max_iterations, memory, gradient_tolerance,
                             relative_objective_tolerance, sufficient_decrease, curvature,
                             max_trials)
        p = np.empty_like(q0)
        reason, iters, evals, tl = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        trace = np.zeros((max_iterations + 1, 6))
        st = L.gs_stats()
        self.check(self.lib.gs_optimize(self.ctx, C.byref(c), C.byref(oc), len(q0), _p(q0), _p(t),
                                        _p(p), C.byref(reason), C.byref(iters), C.byref(evals),
                                        _p(trace), C.byref(tl), C.byref(st)))
        names = ["gradient_tolerance", "objective_tolerance", "max_iterations",
                 "line_search_failure", "non_finite"]
        return {"p0": p, "reason": names[reason.value], "iterations": iters.value,
                "evaluations": evals.value, "trace": trace[:tl.value], "stats": st.as_dict()}

    def optimize_batch(self, q0s, targets, cfg: ShootingConfig, device: int = 0,
                       max_iterations=200, memory=10, gradient_tolerance=1e-6,
                       relative_objective_tolerance=1e-9):
        """Independent registrations (config 5), one stream + host thread each."""
        B = len(q0s)
        q0s = [_arr(q) for q in q0s]
        targets = [_arr(t) for t in targets]
        outs = [np.empty_like(q) for q in q0s]
        c = cfg.c()
        oc = L.gs_opt_config(max_iterations, memory, gradient_tolerance,
                             relative_objective_tolerance, 1e-4, 0.9, 20)
        ns = (C.c_int64 * B)(*[len(q) for q in q0s])
        P = L._d * B
        qa, ta, pa = P(*map(_p, q0s)), P(*map(_p, targets)), P(*map(_p, outs))
        reasons, iters, evals = (C.c_int32 * B)(), (C.c_int32 * B)(), (C.c_int32 * B)()
        tot = np.zeros(B)
        self.check(self.lib.gs_optimize_batch(device, C.byref(c), C.byref(oc), B, ns, qa, ta, pa,
                                              reasons, iters, evals, _p(tot)))
        return {"p0": outs, "reasons": list(reasons), "iterations": list(iters),
                "evaluations": list(evals), "final_total": tot}

    def evaluate_batch(self, q0s, p0s, targets, cfg: ShootingConfig, device: int = 0):
        """Independent evaluations (one stream + host thread each) -> [Evaluation]."""
        B = len(q0s)
        q0s, p0s, targets = ([_arr(a) for a in q0s], [_arr(a) for a in p0s],
                             [_arr(a) for a in targets])
        for q, p, t in zip(q0s, p0s, targets):
            _require_aligned(len(q), len(p), "evaluate_batch")
            _require_aligned(len(q), len(t), "evaluate_batch(target)")
        grads = [np.empty_like(q) for q in q0s]
        c = cfg.c()
        ns = (C.c_int64 * B)(*[len(q) for q in q0s])
        P = L._d * B
        reps, sts = (L.gs_report * B)(), (L.gs_stats * B)()
        self.check(self.lib.gs_evaluate_batch(device, C.byref(c), B, ns, P(*map(_p, q0s)),
                                              P(*map(_p, p0s)), P(*map(_p, targets)), reps,
                                              P(*map(_p, grads)), sts))
        return [Evaluation({"energy": r.energy, "attachment": r.attachment, "total": r.total,
                            "residual_sse": r.residual_sse}, g, s.as_dict())
                for r, g, s in zip(reps, grads, sts)]

    def procrustes_align(self, source, target):
        """procrustes_align (procrustes.cpp:7-58) -> (rotation 3x3, translation, aligned)."""
        s, t = _arr(source, "source"), _arr(target, "target")
        _require_aligned(len(s), len(t), "procrustes_align")
        R, tr, y = np.empty((3, 3)), np.empty(3), np.empty_like(s)
        self.check(self.lib.gs_procrustes_align(self.ctx, len(s), _p(s), _p(t), _p(R), _p(tr), _p(y)))
        return R, tr, y

    def flow(self, cfg: ShootingConfig, n: int) -> "Flow":
        return Flow(self, cfg, n)


class Octree:
    """Device octree (gs_tree); accessors download a host copy on demand."""

    def __init__(self, gs: Geoshoot, handle, q, p):
        self.gs, self.h, self.q, self.p = gs, handle, q, p
        self.n = len(q)
        self._last_m = self.n  # queries of the last call (query_stats)

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.gs.lib.gs_tree_free(self.h)
            self.h = None

    def node_count(self) -> int:
        return self.gs.lib.gs_tree_node_count(self.h)

    def point_count(self) -> int:
        return self.n

    def download(self) -> dict:
        m, n = self.node_count(), self.n
        order = np.empty(n, np.int32)
        kh = np.empty(n, np.uint64)
        kl = np.empty(n, np.uint64)
        level = np.empty(m, np.int32)
        parent = np.empty(m, np.int32)
        skip = np.empty(m, np.int32)
        rng = np.empty((m, 2), np.int32)
        boxes = np.empty((m, 12))
        sums = np.empty((m, 12))
        count = np.empty(m, np.uint32)
        ip = lambda a: a.ctypes.data_as(L._i32p)  # noqa: E731
        self.gs.check(self.gs.lib.gs_tree_download(
            self.h, ip(order), kh.ctypes.data_as(L._u64p), kl.ctypes.data_as(L._u64p), ip(level),
            ip(parent), ip(skip), ip(rng), _p(boxes), _p(sums), count.ctypes.data_as(L._u32p)))
        return {"order": order, "key_hi": kh, "key_lo": kl, "level": level, "parent": parent,
                "skip": skip, "range": rng, "cell_min": boxes[:, 0:3], "cell_max": boxes[:, 3:6],
                "actual_min": boxes[:, 6:9], "actual_max": boxes[:, 9:12],
                "position_sum": sums[:, 0:3], "momentum_sum": sums[:, 3:6],
                "alpha_sum": sums[:, 6:9], "beta_sum": sums[:, 9:12], "count": count}

    def accumulate_adjoints(self, alpha, beta):
        a, b = _arr(alpha), _arr(beta)
        _require_aligned(self.n, len(a), "accumulate_adjoints(alpha)")
        _require_aligned(self.n, len(b), "accumulate_adjoints(beta)")
        self.gs.check(self.gs.lib.gs_tree_accumulate_adjoints(self.h, _p(a), _p(b)))

    def bh_velocity(self, x, sigma, threshold):
        x = _arr(x, "x")
        v = np.empty_like(x)
        st = L.gs_stats()
        self.gs.check(self.gs.lib.gs_bh_velocity(self.h, len(x), _p(x), sigma, threshold, _p(v),
                                                 C.byref(st)))
        self._last_m = len(x)
        return v, st.as_dict()

    def bh_hamiltonian_gradients(self, sigma, threshold):
        dp, dq = np.empty_like(self.q), np.empty_like(self.q)
        st = L.gs_stats()
        self.gs.check(self.gs.lib.gs_bh_rhs(self.h, sigma, threshold, _p(dp), _p(dq),
                                            C.byref(st)))
        self._last_m = self.n
        return dp, dq, st.as_dict()

    def bh_hamiltonian(self, sigma, threshold):
        h = C.c_double()
        st = L.gs_stats()
        self.gs.check(self.gs.lib.gs_bh_hamiltonian(self.h, sigma, threshold, C.byref(h),
                                                    C.byref(st)))
        self._last_m = self.n
        return h.value, st.as_dict()

    def query_stats(self, m=None) -> np.ndarray:
        """Per-query (direct, approximated, visited) counts of the last query call."""
        m = self._last_m if m is None else m
        out = np.empty((m, 3), np.uint64)
        self.gs.check(self.gs.lib.gs_bh_query_stats(self.h, out.ctypes.data_as(L._u64p)))
        return out

    def bh_hessian_products(self, alpha, beta, sigma, threshold):
        a, b = _arr(alpha), _arr(beta)
        out = [np.empty_like(self.q) for _ in range(4)]
        st = L.gs_stats()
        self.gs.check(self.gs.lib.gs_bh_hessian_products(self.h, _p(a), _p(b), sigma, threshold,
                                                         *map(_p, out), C.byref(st)))
        self._last_m = self.n
        return tuple(out) + (st.as_dict(),)

    def bh_point_gradients(self, x, px, sigma, threshold):
        """bh_point_gradients (bh_kernel.cpp:81-112) at m arbitrary (x, px)."""
        x, px = _arr(x, "x"), _arr(px, "px")
        _require_aligned(len(x), len(px), "bh_point_gradients")
        dp, dq = np.empty_like(x), np.empty_like(x)
        st = L.gs_stats()
        self.gs.check(self.gs.lib.gs_bh_point_gradients(self.h, len(x), _p(x), _p(px), sigma,
                                                        threshold, _p(dp), _p(dq), C.byref(st)))
        self._last_m = len(x)
        return dp, dq, st.as_dict()

    def bh_point_hessian_products(self, qi, pi, alpha_i, beta_i, alpha, beta, sigma, threshold):
        """bh_point_hessian_products (bh_kernel.cpp:114-160) at m arbitrary queries;
        alpha/beta (n x 3, or None) are the per-point adjoints of the direct terms."""
        qi, pi, ai, bi = (_arr(v) for v in (qi, pi, alpha_i, beta_i))
        m = len(qi)
        for v, nm in ((pi, "pi"), (ai, "alpha_i"), (bi, "beta_i")):
            _require_aligned(m, len(v), f"bh_point_hessian_products({nm})")
        a = None if alpha is None else _arr(alpha)
        b = None if beta is None else _arr(beta)
        out = [np.empty_like(qi) for _ in range(4)]
        st = L.gs_stats()
        self.gs.check(self.gs.lib.gs_bh_point_hessian_products(
            self.h, m, _p(qi), _p(pi), _p(ai), _p(bi), _p(a), _p(b), sigma, threshold,
            *map(_p, out), C.byref(st)))
        self._last_m = m
        return tuple(out) + (st.as_dict(),)


class Flow:
    """Device-resident flow (gs_flow): (q, p) stay in HBM between advances."""

    def __init__(self, gs: Geoshoot, cfg: ShootingConfig, n: int):
        self.gs, self.cfg, self.n = gs, cfg, n
        self._c = cfg.c()
        h = C.c_void_p()
        gs.check(gs.lib.gs_flow_create(gs.ctx, C.byref(self._c), n, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.gs.lib.gs_flow_destroy(self.h)
            self.h = None

    def upload(self, q0, p0):
        q0, p0 = _arr(q0), _arr(p0)
        self.gs.check(self.gs.lib.gs_flow_upload(self.h, _p(q0), _p(p0)))

    def advance(self, steps: int):
        self.gs.check(self.gs.lib.gs_flow_advance(self.h, steps))

    def sync(self):
        self.gs.check(self.gs.lib.gs_flow_sync(self.h))

    def download(self):
        q, p = np.empty((self.n, 3)), np.empty((self.n, 3))
        self.gs.check(self.gs.lib.gs_flow_download(self.h, _p(q), _p(p)))
        return q, p

    def last_launches(self) -> int:
        return self.gs.lib.gs_flow_last_launches(self.h)

    def stats(self) -> dict:
        st = L.gs_stats()
        self.gs.check(self.gs.lib.gs_flow_stats(self.h, C.byref(st)))
        return st.as_dict()

    def stream(self) -> int:
        return self.gs.lib.gs_flow_stream(self.h) or 0

    def profile(self, enable: bool = True):
        self.gs.check(self.gs.lib.gs_flow_profile(self.h, 1 if enable else 0))

    def profile_read(self):
        k, b = C.c_double(), C.c_double()
        kl, bl = C.c_int64(), C.c_int64()
        self.gs.check(self.gs.lib.gs_flow_profile_read(self.h, C.byref(k), C.byref(kl), C.byref(b),
                                                       C.byref(bl)))
        return {"kernel_ms": k.value, "kernel_launches": kl.value, "build_ms": b.value,
                "builds": bl.value}

    def profile_phases(self, channels: int = 6):
        import numpy as _np
        ms = _np.zeros(channels)
        cnt = _np.zeros(channels, _np.int64)
        self.gs.check(self.gs.lib.gs_flow_profile_phases(
            self.h, _p(ms), cnt.ctypes.data_as(C.POINTER(C.c_int64)), channels))
        names = ["kernel", "build", "bbox_keys", "sort", "topology", "aggregate", "c6", "c7"]
        return {names[c]: {"ms": float(ms[c]), "count": int(cnt[c])} for c in range(channels)}

    # sharded stage API (see shard.py)
    def set_shard(self, begin: int, count: int):
        self.gs.check(self.gs.lib.gs_flow_set_shard(self.h, begin, count))

    def source_buffer(self) -> int:
        return self.gs.lib.gs_flow_source_buffer(self.h) or 0

    def record_bytes(self) -> int:
        return self.gs.lib.gs_flow_record_bytes(self.h)

    def stage(self, s: int):
        self.gs.check(self.gs.lib.gs_flow_stage(self.h, s))

    # ---- multi-GPU symmetric exact stages (gs_flow_set_pair_rows) ------------
    def set_pair_rows(self, rank: int, world: int) -> bool:
        """Use this rank's rows of the symmetric tile-pair grid for the exact
        RHS (False: the flow does not qualify; stage() stays the path)."""
        en = C.c_int32()
        self.gs.check(self.gs.lib.gs_flow_set_pair_rows(self.h, rank, world, C.byref(en)))
        return bool(en.value)

    def stage_pairs(self, s: int) -> int:
        """This rank's rows for stage s, folded per target: device pointer to
        n x 8 float32 partials {A.xyz, 0, B.xyz, 0} (valid until the next call)."""
        ptr = C.c_void_p()
        self.gs.check(self.gs.lib.gs_flow_stage_pairs(self.h, s, C.byref(ptr)))
        return ptr.value or 0

    def stage_apply(self, s: int, partials_ptr: int, nparts: int):
        """The shard's stage epilogue over nparts partials [part][shard] x 8 float32."""
        self.gs.check(self.gs.lib.gs_flow_stage_apply(self.h, s, C.c_void_p(partials_ptr), nparts))
