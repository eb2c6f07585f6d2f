"""Seeded synthetic inputs (BASELINE.json configs) and metrics."""
import numpy as np


def rel_l2(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    den = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / (den if den > 0 else 1.0))


def f32(a):
    """Round to FP32 and promote back: the inputs the FP32 path really sees."""
    return np.asarray(a, np.float32).astype(np.float64)


def uniform(n, extent=1.0, seed=0):
    return np.random.default_rng(seed).uniform(0.0, extent, (n, 3))


def sym_uniform(n, scale=1.0, seed=0):
    return np.random.default_rng(seed).uniform(-scale, scale, (n, 3))


def sphere(n, seed=0):
    """C1: Archimedes sampling on the unit sphere."""
    rng = np.random.default_rng(seed)
    z = rng.uniform(-1, 1, n)
    t = rng.uniform(0, 2 * np.pi, n)
    r = np.sqrt(1 - z * z)
    return np.stack([r * np.cos(t), r * np.sin(t), z], 1)


def ellipsoid(n, axes=(30.0, 15.0, 10.0), jitter=0.5, seed=0):
    """C2: area-uniform on an ellipsoid (rejection) + isotropic normal jitter."""
    rng = np.random.default_rng(seed)
    a, b, c = axes
    out = []
    gmax = max(b * c, a * c, a * b)
    while sum(len(o) for o in out) < n:
        m = 2 * n
        z = rng.uniform(-1, 1, m)
        t = rng.uniform(0, 2 * np.pi, m)
        r = np.sqrt(1 - z * z)
        u = np.stack([r * np.cos(t), r * np.sin(t), z], 1)
        g = np.sqrt((b * c * u[:, 0]) ** 2 + (a * c * u[:, 1]) ** 2 + (a * b * u[:, 2]) ** 2)
        keep = rng.uniform(0, gmax, m) < g
        out.append(u[keep] * np.array([a, b, c]))
    q = np.concatenate(out)[:n]
    return q + rng.normal(0, jitter, q.shape)


def smooth_momenta(q, amp, seed=0, k=4, wlen=0.1):
    """p_c(q) = amp * sum_k sin(q . w_k + phi_kc), |w_k| = wlen."""
    rng = np.random.default_rng(seed)
    w = rng.normal(size=(k, 3))
    w = wlen * w / np.linalg.norm(w, axis=1, keepdims=True)
    phi = rng.uniform(0, 2 * np.pi, (k, 3))
    return amp * np.sin((q @ w.T)[:, :, None] + phi[None]).sum(1)


def tube(n, R=40.0, r=4.0, span=2 * np.pi / 3, seed=0):
    """C3: area-uniform tube surface around a circular arc."""
    rng = np.random.default_rng(seed)
    out = []
    while sum(len(o) for o in out) < n:
        m = 2 * n
        s = rng.uniform(0, span, m)
        t = rng.uniform(0, 2 * np.pi, m)
        keep = rng.uniform(0, 1, m) < (R + r * np.cos(t)) / (R + r)
        s, t = s[keep], t[keep]
        out.append(np.stack([(R + r * np.cos(t)) * np.cos(s), (R + r * np.cos(t)) * np.sin(s),
                             r * np.sin(t)], 1))
    return np.concatenate(out)[:n]
