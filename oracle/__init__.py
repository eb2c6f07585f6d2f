"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the two CPU checkers.

* ``port``: our plain-C restatement of the reference hot path (oracle/port.c),
  built here and on the GPU box by ``make -C oracle port``.
* ``ref``:  the UNMODIFIED reference sources compiled by path
  (oracle/Makefile -> oracle/_ref/libgeoshoot_ref.so), built in the container
  that holds /root/reference and shipped prebuilt to the GPU box.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package; the
product (``paper_1907_04834_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle_port.so")
REF_SO = os.path.join(HERE, "_ref", "libgeoshoot_ref.so")
# built with -DGEOSHOOT_BH_LITERAL_MEAN_DOT (oracle/Makefile): literal_mean_dot parity
REF_LMD_SO = os.path.join(HERE, "_ref", "libgeoshoot_ref_lmd.so")

_d = C.POINTER(C.c_double)
_u64 = C.POINTER(C.c_uint64)
_i32 = C.POINTER(C.c_int32)
_i64 = C.c_int64


def _p(a):
    return None if a is None else a.ctypes.data_as(_d)


def _vec(n):
    return np.zeros((n, 3), dtype=np.float64)


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, status, step=0):
        super().__init__(f"oracle status {status} (step {step})")
        self.status = status
        self.step = step


# --------------------------------------------------------------------------
class Port:
    """C restatement (oracle/port.c)."""

    def __init__(self, path=PORT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle port`")
        L = self.lib = C.CDLL(path)
        L.port_hamiltonian.restype = C.c_double
        L.port_hamiltonian.argtypes = [_i64, _d, _d, C.c_double]
        L.port_exact_rhs.restype = C.c_double
        L.port_exact_rhs.argtypes = [_i64, _d, _d, C.c_double, _d, _d]
        L.port_exact_velocity.argtypes = [_i64, _d, _i64, _d, _d, C.c_double, _d]
        L.port_hessian_products.argtypes = [_i64, _d, _d, _d, _d, C.c_double, _d, _d, _d, _d]
        L.port_tree_build.restype = C.c_void_p
        L.port_tree_build.argtypes = [_i64, _d, _d]
        L.port_tree_free.argtypes = [C.c_void_p]
        L.port_tree_node_count.restype = _i64
        L.port_tree_node_count.argtypes = [C.c_void_p]
        L.port_tree_dump.argtypes = [C.c_void_p, _d, _d, _i32, _i32]
        L.port_tree_accumulate.argtypes = [C.c_void_p, _d, _d]
        L.port_tree_leaf_order.argtypes = [C.c_void_p, _i32]
        L.port_root_box.argtypes = [_i64, _d, _d, _d]
        L.port_morton_keys.argtypes = [_i64, _d, _d, _d, _u64, _u64]
        L.port_bh_rhs.argtypes = [C.c_void_p, _i64, _d, _d, C.c_double, C.c_double, C.c_int, _d, _d, _u64]
        L.port_bh_hessprod.argtypes = [C.c_void_p, _i64, _d, _d, _d, _d, C.c_double, C.c_double,
                                       C.c_int, _d, _d, _d, _d]
        L.port_bh_velocity.argtypes = [C.c_void_p, _i64, _d, C.c_double, C.c_double, C.c_int, _d, _u64]
        L.port_shoot_forward.restype = C.c_int
        L.port_shoot_forward.argtypes = [_i64, _d, _d, C.c_double, C.c_int, C.c_int, C.c_double,
                                         C.c_int, C.c_int, _d, _d, _d, _d, _d, C.POINTER(C.c_int)]
        L.port_evaluate.restype = C.c_int
        L.port_evaluate.argtypes = [_i64, _d, _d, _d, C.c_double, C.c_double, C.c_int, C.c_int,
                                    C.c_double, C.c_int, _d, _d, C.POINTER(C.c_int)]
        L.port_warp.restype = C.c_int
        L.port_warp.argtypes = [_i64, C.c_int, _d, _d, _i64, _d, C.c_double, C.c_int, C.c_double,
                                C.c_int, _d, C.POINTER(C.c_int)]

    # kernel_exact ---------------------------------------------------------
    def hamiltonian(self, q, p, sigma):
        q, p = _c(q), _c(p)
        return self.lib.port_hamiltonian(len(q), _p(q), _p(p), sigma)

    def exact_rhs(self, q, p, sigma):
        q, p = _c(q), _c(p)
        dp, dq = _vec(len(q)), _vec(len(q))
        h = self.lib.port_exact_rhs(len(q), _p(q), _p(p), sigma, _p(dp), _p(dq))
        return dp, dq, h

    def exact_velocity(self, x, q, p, sigma):
        x, q, p = _c(x), _c(q), _c(p)
        v = _vec(len(x))
        self.lib.port_exact_velocity(len(x), _p(x), len(q), _p(q), _p(p), sigma, _p(v))
        return v

    def hessian_products(self, q, p, alpha, beta, sigma):
        q, p, a, b = _c(q), _c(p), _c(alpha), _c(beta)
        out = [_vec(len(q)) for _ in range(4)]
        self.lib.port_hessian_products(len(q), _p(q), _p(p), _p(a), _p(b), sigma, *map(_p, out))
        return tuple(out)

    # octree ---------------------------------------------------------------
    def tree(self, q, p):
        return PortTree(self, _c(q), _c(p))

    def root_box(self, q):
        q = _c(q)
        lo, hi = np.zeros(3), np.zeros(3)
        self.lib.port_root_box(len(q), _p(q), _p(lo), _p(hi))
        return lo, hi

    def morton_keys(self, q, lo=None, hi=None):
        q = _c(q)
        if lo is None:
            lo, hi = self.root_box(q)
        kh = np.zeros(len(q), np.uint64)
        kl = np.zeros(len(q), np.uint64)
        self.lib.port_morton_keys(len(q), _p(q), _p(_c(lo)), _p(_c(hi)),
                                  kh.ctypes.data_as(_u64), kl.ctypes.data_as(_u64))
        return kh, kl

    # shooting -------------------------------------------------------------
    def shoot_forward(self, q0, p0, sigma, timesteps, backend=0, thr_mult=3.0,
                      integrator=0, threads=0, keep_traj=True):
        q0, p0 = _c(q0), _c(p0)
        n = len(q0)
        threads = threads or os.cpu_count() or 1
        tq = np.zeros((timesteps + 1, n, 3)) if keep_traj else None
        tp = np.zeros((timesteps + 1, n, 3)) if keep_traj else None
        fq, fp = _vec(n), _vec(n)
        e = C.c_double(0.0)
        bad = C.c_int(0)
        st = self.lib.port_shoot_forward(n, _p(q0), _p(p0), sigma, timesteps, backend, thr_mult,
                                         integrator, threads, _p(tq), _p(tp), _p(fq), _p(fp),
                                         C.byref(e), C.byref(bad))
        if st:
            raise OracleError(st, bad.value)
        return {"q": fq, "p": fp, "energy": e.value, "traj_q": tq, "traj_p": tp}

    def evaluate(self, q0, p0, target, sigma, lam, timesteps, backend=0, thr_mult=3.0, threads=0):
        q0, p0, t = _c(q0), _c(p0), _c(target)
        n = len(q0)
        rep = np.zeros(4)
        g = _vec(n)
        bad = C.c_int(0)
        st = self.lib.port_evaluate(n, _p(q0), _p(p0), _p(t), sigma, lam, timesteps, backend,
                                    thr_mult, threads or os.cpu_count() or 1, _p(rep), _p(g),
                                    C.byref(bad))
        if st:
            raise OracleError(st, bad.value)
        return rep, g

    def warp(self, traj_q, traj_p, x, sigma, backend=0, thr_mult=3.0, threads=0):
        tq, tp, x = _c(traj_q), _c(traj_p), _c(x)
        y = _vec(len(x))
        bad = C.c_int(0)
        st = self.lib.port_warp(tq.shape[1], tq.shape[0] - 1, _p(tq), _p(tp), len(x), _p(x),
                                sigma, backend, thr_mult, threads or os.cpu_count() or 1, _p(y),
                                C.byref(bad))
        if st:
            raise OracleError(st, bad.value)
        return y


class _TreeDump:
    def dump(self):
        m = self.node_count()
        boxes = np.zeros((m, 12))
        sums = np.zeros((m, 12))
        ints = np.zeros((m, 11), np.int32)
        nxt = np.zeros(self.n, np.int32)
        self._dump(boxes.ctypes.data_as(_d), sums.ctypes.data_as(_d),
                   ints.ctypes.data_as(_i32), nxt.ctypes.data_as(_i32))
        return {
            "cell_min": boxes[:, 0:3], "cell_max": boxes[:, 3:6],
            "actual_min": boxes[:, 6:9], "actual_max": boxes[:, 9:12],
            "position_sum": sums[:, 0:3], "momentum_sum": sums[:, 3:6],
            "alpha_sum": sums[:, 6:9], "beta_sum": sums[:, 9:12],
            "count": ints[:, 0].copy(), "children": ints[:, 1:9].copy(),
            "first_point": ints[:, 9].copy(), "leaf": ints[:, 10].astype(bool),
            "next_point": nxt,
        }


class PortTree(_TreeDump):
    def __init__(self, port, q, p):
        self.port, self.n = port, len(q)
        self.q, self.p = q, p
        self.h = port.lib.port_tree_build(len(q), _p(q), _p(p))

    def __del__(self):
        if getattr(self, "h", None):
            self.port.lib.port_tree_free(self.h)
            self.h = None

    def node_count(self):
        return self.port.lib.port_tree_node_count(self.h)

    def _dump(self, *a):
        self.port.lib.port_tree_dump(self.h, *a)

    def accumulate(self, alpha, beta):
        a, b = _c(alpha), _c(beta)
        self.port.lib.port_tree_accumulate(self.h, _p(a), _p(b))

    def leaf_order(self):
        o = np.zeros(self.n, np.int32)
        self.port.lib.port_tree_leaf_order(self.h, o.ctypes.data_as(_i32))
        return o

    def bh_rhs(self, sigma, thr, threads=0, q=None, p=None):
        q = self.q if q is None else _c(q)
        p = self.p if p is None else _c(p)
        dp, dq = _vec(len(q)), _vec(len(q))
        pq = np.zeros((len(q), 3), np.uint64)
        self.port.lib.port_bh_rhs(self.h, len(q), _p(q), _p(p), sigma, thr,
                                  threads or os.cpu_count() or 1, _p(dp), _p(dq),
                                  pq.ctypes.data_as(_u64))
        return dp, dq, pq

    def bh_hessprod(self, alpha, beta, sigma, thr, threads=0):
        a, b = _c(alpha), _c(beta)
        out = [_vec(self.n) for _ in range(4)]
        self.port.lib.port_bh_hessprod(self.h, self.n, _p(self.q), _p(self.p), _p(a), _p(b),
                                       sigma, thr, threads or os.cpu_count() or 1, *map(_p, out))
        return tuple(out)

    def bh_velocity(self, x, sigma, thr, threads=0):
        x = _c(x)
        v = _vec(len(x))
        pq = np.zeros((len(x), 3), np.uint64)
        self.port.lib.port_bh_velocity(self.h, len(x), _p(x), sigma, thr,
                                       threads or os.cpu_count() or 1, _p(v),
                                       pq.ctypes.data_as(_u64))
        return v, pq


# --------------------------------------------------------------------------
class Ref:
    """The reference's own sources compiled by path (oracle/_ref)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = self.lib = C.CDLL(path)
        for name, args in {
            "ref_hamiltonian": [_i64, _d, _d, C.c_double, _d],
            "ref_exact_rhs": [_i64, _d, _d, C.c_double, _d, _d, _d],
            "ref_exact_rhs_concurrent": [_i64, _d, _d, C.c_double, C.c_int, C.c_int, _d, _d],
            "ref_exact_velocity": [_i64, _d, _i64, _d, _d, C.c_double, _d],
            "ref_hessian_products": [_i64, _d, _d, _d, _d, C.c_double, _d, _d, _d, _d],
            "ref_tree_accumulate": [C.c_void_p, _i64, _d, _d],
            "ref_bh_velocity": [C.c_void_p, _i64, _d, C.c_double, C.c_double, _d, _u64],
            "ref_bh_rhs": [C.c_void_p, _i64, _d, _d, C.c_double, C.c_double, C.c_int, _d, _d, _u64],
            "ref_bh_hessprod": [C.c_void_p, _i64, _d, _d, _d, _d, C.c_double, C.c_double, C.c_int,
                                _d, _d, _d, _d, _u64],
            "ref_bh_point_gradients": [C.c_void_p, _i64, _d, _d, C.c_double, C.c_double, C.c_int,
                                       _d, _d, _u64],
            "ref_bh_point_hessprod": [C.c_void_p, _i64, _d, _d, _d, _d, _i64, _d, _d, C.c_double,
                                      C.c_double, C.c_int, _d, _d, _d, _d, _u64],
            "ref_bh_velocity_pq": [C.c_void_p, _i64, _d, C.c_double, C.c_double, C.c_int, _d, _u64],
            "ref_bh_hamiltonian": [C.c_void_p, _i64, _d, _d, C.c_double, C.c_double, _d],
            "ref_shoot_forward": [_i64, _d, _d, C.c_double, C.c_int, C.c_int, C.c_double, _d, _d],
            "ref_objective": [_i64, _d, _d, _d, C.c_double, C.c_double, C.c_int, C.c_int,
                              C.c_double, _d],
            "ref_evaluate": [_i64, _d, _d, _d, C.c_double, C.c_double, C.c_int, C.c_int,
                             C.c_double, C.c_int, _d, _d, _u64, _d],
            "ref_backward_gradient": [_i64, C.c_int, _d, _d, _d, C.c_double, C.c_double, C.c_int,
                                      C.c_int, C.c_double, _d],
            "ref_warp_points": [_i64, C.c_int, _d, _d, _i64, _d, C.c_double, C.c_int, C.c_int,
                                C.c_double, _d],
            "ref_generate": [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64, _d],
            "ref_read_points": [C.c_char_p, C.c_int, _d, _i64, C.POINTER(_i64),
                                C.POINTER(C.c_longlong)],
            "ref_write_points": [C.c_char_p, C.c_int, _i64, _d, C.c_char_p],
            "ref_optimize": [_i64, _d, _d, C.c_double, C.c_double, C.c_int, C.c_int, C.c_double,
                             C.c_int, _d, C.POINTER(C.c_int), C.POINTER(C.c_int), _d,
                             C.POINTER(C.c_int)],
        }.items():
            getattr(L, name).argtypes = args
            getattr(L, name).restype = C.c_int
        L.ref_tree_build.restype = C.c_void_p
        L.ref_tree_build.argtypes = [_i64, _d, _d, C.POINTER(C.c_int)]
        L.ref_tree_free.argtypes = [C.c_void_p]
        L.ref_tree_node_count.restype = _i64
        L.ref_tree_node_count.argtypes = [C.c_void_p]
        L.ref_tree_dump.argtypes = [C.c_void_p, _d, _d, _i32, _i32]
        L.ref_validate_config.restype = C.c_uint
        L.ref_validate_config.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double]
        L.ref_last_nonfinite_step.restype = C.c_int

    def _chk(self, st):
        if st:
            raise OracleError(st, self.lib.ref_last_nonfinite_step())

    def hamiltonian(self, q, p, sigma):
        q, p = _c(q), _c(p)
        h = C.c_double()
        self._chk(self.lib.ref_hamiltonian(len(q), _p(q), _p(p), sigma, C.byref(h)))
        return h.value

    def exact_rhs(self, q, p, sigma):
        q, p = _c(q), _c(p)
        dp, dq = _vec(len(q)), _vec(len(q))
        h = C.c_double()
        self._chk(self.lib.ref_exact_rhs(len(q), _p(q), _p(p), sigma, _p(dp), _p(dq), C.byref(h)))
        return dp, dq, h.value

    def exact_rhs_concurrent(self, q, p, sigma, threads, reps=1):
        q, p = _c(q), _c(p)
        dp, dq = _vec(len(q)), _vec(len(q))
        self._chk(self.lib.ref_exact_rhs_concurrent(len(q), _p(q), _p(p), sigma, threads, reps,
                                                    _p(dp), _p(dq)))
        return dp, dq

    def exact_velocity(self, x, q, p, sigma):
        x, q, p = _c(x), _c(q), _c(p)
        v = _vec(len(x))
        self._chk(self.lib.ref_exact_velocity(len(x), _p(x), len(q), _p(q), _p(p), sigma, _p(v)))
        return v

    def hessian_products(self, q, p, alpha, beta, sigma):
        q, p, a, b = _c(q), _c(p), _c(alpha), _c(beta)
        out = [_vec(len(q)) for _ in range(4)]
        self._chk(self.lib.ref_hessian_products(len(q), _p(q), _p(p), _p(a), _p(b), sigma,
                                                *map(_p, out)))
        return tuple(out)

    def tree(self, q, p):
        return RefTree(self, _c(q), _c(p))

    def shoot_forward(self, q0, p0, sigma, timesteps, backend=0, thr_mult=3.0):
        q0, p0 = _c(q0), _c(p0)
        n = len(q0)
        tq = np.zeros((timesteps + 1, n, 3))
        tp = np.zeros((timesteps + 1, n, 3))
        self._chk(self.lib.ref_shoot_forward(n, _p(q0), _p(p0), sigma, timesteps, backend,
                                             thr_mult, _p(tq), _p(tp)))
        return tq, tp

    def objective(self, q0, p0, target, sigma, lam, timesteps, backend=0, thr_mult=3.0):
        q0, p0, t = _c(q0), _c(p0), _c(target)
        rep = np.zeros(4)
        self._chk(self.lib.ref_objective(len(q0), _p(q0), _p(p0), _p(t), sigma, lam, timesteps,
                                         backend, thr_mult, _p(rep)))
        return rep

    def evaluate(self, q0, p0, target, sigma, lam, timesteps, backend=0, thr_mult=3.0, threads=0):
        q0, p0, t = _c(q0), _c(p0), _c(target)
        rep = np.zeros(4)
        g = _vec(len(q0))
        stats = np.zeros(4, np.uint64)
        times = np.zeros(3)
        self._chk(self.lib.ref_evaluate(len(q0), _p(q0), _p(p0), _p(t), sigma, lam, timesteps,
                                        backend, thr_mult, threads, _p(rep), _p(g),
                                        stats.ctypes.data_as(_u64), _p(times)))
        return rep, g, stats, times

    def backward_gradient(self, traj_q, traj_p, target, sigma, lam, timesteps, backend=0,
                          thr_mult=3.0):
        tq, tp, t = _c(traj_q), _c(traj_p), _c(target)
        g = _vec(tq.shape[1])
        self._chk(self.lib.ref_backward_gradient(tq.shape[1], tq.shape[0], _p(tq), _p(tp), _p(t),
                                                 sigma, lam, timesteps, backend, thr_mult, _p(g)))
        return g

    def warp_points(self, traj_q, traj_p, x, sigma, timesteps, backend=0, thr_mult=3.0):
        tq, tp, x = _c(traj_q), _c(traj_p), _c(x)
        y = _vec(len(x))
        self._chk(self.lib.ref_warp_points(tq.shape[1], tq.shape[0], _p(tq), _p(tp), len(x), _p(x),
                                           sigma, timesteps, backend, thr_mult, _p(y)))
        return y

    def optimize(self, q0, target, sigma, lam, timesteps, backend=0, thr_mult=3.0,
                 max_iterations=200):
        q0, t = _c(q0), _c(target)
        p = _vec(len(q0))
        reason, iters, tl = C.c_int(), C.c_int(), C.c_int()
        trace = np.zeros((max_iterations + 1, 6))
        self._chk(self.lib.ref_optimize(len(q0), _p(q0), _p(t), sigma, lam, timesteps, backend,
                                        thr_mult, max_iterations, _p(p), C.byref(reason),
                                        C.byref(iters), _p(trace), C.byref(tl)))
        names = ["gradient_tolerance", "objective_tolerance", "max_iterations",
                 "line_search_failure", "non_finite"]
        return {"p0": p, "reason": names[reason.value], "iterations": iters.value,
                "trace": trace[:tl.value]}

    def read_points(self, path, vtk):
        """-> (status, points or None, parse line). The reference's iostream
        parsing crashes inside a process that has imported numpy (observed),
        so it runs in a numpy-free child process."""
        import json
        import subprocess
        import sys
        code = (
            "import ctypes as C, json, sys\n"
            "L = C.CDLL(sys.argv[1])\n"
            "L.ref_read_points.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_double), C.c_int64,"
            " C.POINTER(C.c_int64), C.POINTER(C.c_longlong)]\n"
            "n, line = C.c_int64(), C.c_longlong()\n"
            "st = L.ref_read_points(sys.argv[2].encode(), int(sys.argv[3]), None, 0, C.byref(n), C.byref(line))\n"
            "pts = None\n"
            "if st == 0:\n"
            "    buf = (C.c_double * (3 * n.value))()\n"
            "    L.ref_read_points(sys.argv[2].encode(), int(sys.argv[3]), buf, n.value, C.byref(n), C.byref(line))\n"
            "    pts = [float.hex(v) for v in buf]\n"
            "print(json.dumps([st, line.value, pts]))\n")
        out = subprocess.run([sys.executable, "-c", code, REF_SO, path, str(int(vtk))],
                             capture_output=True, text=True, check=True).stdout
        st, line, pts = json.loads(out)
        if st:
            return st, None, line
        return 0, np.array([float.fromhex(v) for v in pts]).reshape(-1, 3), 0

    def write_points(self, path, vtk, pts, header=None):
        pts = _c(pts)
        self._chk(self.lib.ref_write_points(path.encode(), vtk, len(pts), _p(pts),
                                            header.encode() if header else None))

    def validate_config(self, sigma, lam, timesteps, thr_mult):
        return self.lib.ref_validate_config(sigma, lam, timesteps, thr_mult)

    def generate(self, kind, n, a=0.0, b=0.0, c=0.0, seed=0):
        out = _vec(n)
        self._chk(self.lib.ref_generate(kind, n, a, b, c, seed, _p(out)))
        return out


class RefTree(_TreeDump):
    def __init__(self, ref, q, p):
        self.ref, self.n, self.q, self.p = ref, len(q), q, p
        st = C.c_int(0)
        self.h = ref.lib.ref_tree_build(len(q), _p(q), _p(p), C.byref(st))
        if st.value:
            self.h = None
            raise OracleError(st.value)

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_tree_free(self.h)
            self.h = None

    def node_count(self):
        return self.ref.lib.ref_tree_node_count(self.h)

    def _dump(self, *a):
        self.ref.lib.ref_tree_dump(self.h, *a)

    def accumulate(self, alpha, beta):
        a, b = _c(alpha), _c(beta)
        self.ref._chk(self.ref.lib.ref_tree_accumulate(self.h, self.n, _p(a), _p(b)))

    def bh_rhs(self, sigma, thr, threads=0):
        dp, dq = _vec(self.n), _vec(self.n)
        pq = np.zeros((self.n, 3), np.uint64)
        self.ref._chk(self.ref.lib.ref_bh_rhs(self.h, self.n, _p(self.q), _p(self.p), sigma, thr,
                                              threads, _p(dp), _p(dq), pq.ctypes.data_as(_u64)))
        return dp, dq, pq

    def bh_hessprod(self, alpha, beta, sigma, thr, threads=0, per_query=False):
        a, b = _c(alpha), _c(beta)
        out = [_vec(self.n) for _ in range(4)]
        pq = np.zeros((self.n, 3), np.uint64)
        self.ref._chk(self.ref.lib.ref_bh_hessprod(self.h, self.n, _p(self.q), _p(self.p), _p(a),
                                                   _p(b), sigma, thr, threads, *map(_p, out),
                                                   pq.ctypes.data_as(_u64)))
        return tuple(out) + ((pq,) if per_query else ())

    def bh_point_gradients(self, x, px, sigma, thr, threads=0):
        x, px = _c(x), _c(px)
        dp, dq = _vec(len(x)), _vec(len(x))
        pq = np.zeros((len(x), 3), np.uint64)
        self.ref._chk(self.ref.lib.ref_bh_point_gradients(self.h, len(x), _p(x), _p(px), sigma,
                                                          thr, threads, _p(dp), _p(dq),
                                                          pq.ctypes.data_as(_u64)))
        return dp, dq, pq

    def bh_point_hessprod(self, qi, pi, ai, bi, alpha, beta, sigma, thr, threads=0):
        qi, pi, ai, bi, a, b = (_c(v) for v in (qi, pi, ai, bi, alpha, beta))
        out = [_vec(len(qi)) for _ in range(4)]
        pq = np.zeros((len(qi), 3), np.uint64)
        self.ref._chk(self.ref.lib.ref_bh_point_hessprod(
            self.h, len(qi), _p(qi), _p(pi), _p(ai), _p(bi), len(a), _p(a), _p(b), sigma, thr,
            threads, *map(_p, out), pq.ctypes.data_as(_u64)))
        return tuple(out) + (pq,)

    def bh_velocity_pq(self, x, sigma, thr, threads=0):
        x = _c(x)
        v = _vec(len(x))
        pq = np.zeros((len(x), 3), np.uint64)
        self.ref._chk(self.ref.lib.ref_bh_velocity_pq(self.h, len(x), _p(x), sigma, thr, threads,
                                                      _p(v), pq.ctypes.data_as(_u64)))
        return v, pq

    def bh_hamiltonian(self, sigma, thr):
        h = C.c_double()
        self.ref._chk(self.ref.lib.ref_bh_hamiltonian(self.h, self.n, _p(self.q), _p(self.p), sigma,
                                                      thr, C.byref(h)))
        return h.value

    def bh_velocity(self, x, sigma, thr):
        x = _c(x)
        v = _vec(len(x))
        stats = np.zeros(3, np.uint64)
        self.ref._chk(self.ref.lib.ref_bh_velocity(self.h, len(x), _p(x), sigma, thr, _p(v),
                                                   stats.ctypes.data_as(_u64)))
        return v, stats


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref


def have_ref() -> bool:
    return os.path.exists(REF_SO)


_ref_lmd = None


def ref_lmd() -> Ref:
    """The reference built with GEOSHOOT_BH_LITERAL_MEAN_DOT (aggregate dot scale 1/count)."""
    global _ref_lmd
    if _ref_lmd is None:
        _ref_lmd = Ref(REF_LMD_SO)
    return _ref_lmd
