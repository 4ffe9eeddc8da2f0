"""Quaternion algebra for material frames (host side, numpy).

Scalar-first unit quaternions q = (w, x, y, z) rotate body vectors into the
world frame; the third column of R(q) is the director d3 that the
quaternion-tangent penalty aligns with the centreline tangent.

Mirrors the reference helper module (rodsim/quat.py:1-119): same names,
same conventions.  The device kernels restate these formulas with the
reference compiled core's operation order (csrc/rod_math.cuh).
"""

import numpy as np

IDENTITY = np.array([1.0, 0.0, 0.0, 0.0])


def _as(q):
    return np.asarray(q, dtype=float)


def multiply(a, b):
    """Hamilton product a*b over the last axis (broadcasting)."""
    a, b = _as(a), _as(b)
    a0, a1, a2, a3 = np.moveaxis(a, -1, 0)
    b0, b1, b2, b3 = np.moveaxis(b, -1, 0)
    return np.stack([
        a0 * b0 - a1 * b1 - a2 * b2 - a3 * b3,
        a0 * b1 + b0 * a1 + a2 * b3 - a3 * b2,
        a0 * b2 + b0 * a2 + a3 * b1 - a1 * b3,
        a0 * b3 + b0 * a3 + a1 * b2 - a2 * b1,
    ], axis=-1)


def conjugate(q):
    out = _as(q).copy()
    out[..., 1:] = -out[..., 1:]
    return out


def normalize(q):
    q = _as(q)
    return q / np.linalg.norm(q, axis=-1, keepdims=True)


def from_axis_angle(axis, angle):
    axis = _as(axis)
    axis = axis / np.linalg.norm(axis)
    h = 0.5 * angle
    return np.concatenate([[np.cos(h)], np.sin(h) * axis])


def rotate(q, v):
    """World-frame image of body vector(s) v."""
    v = _as(v)
    pure = np.concatenate([np.zeros(v.shape[:-1] + (1,)), v], axis=-1)
    return multiply(multiply(q, pure), conjugate(q))[..., 1:]


def director3(q):
    """d3(q): third column of R(q), kept as an unnormalised polynomial."""
    q = _as(q)
    w, x, y, z = np.moveaxis(q, -1, 0)
    return np.stack([2.0 * (x * z + w * y),
                     2.0 * (y * z - w * x),
                     1.0 - 2.0 * (x * x + y * y)], axis=-1)


def director3_jacobian(q):
    """d d3 / d q with shape (..., 3, 4)."""
    q = _as(q)
    w, x, y, z = np.moveaxis(q, -1, 0)
    zero = np.zeros_like(w)
    rows = [[2 * y, 2 * z, 2 * w, 2 * x],
            [-2 * x, -2 * w, 2 * z, 2 * y],
            [zero, -4 * x, -4 * y, zero]]
    return np.stack([np.stack(r, axis=-1) for r in rows], axis=-2)


def to_matrix(q):
    w, x, y, z = _as(q)
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])


def _skew_form(pairs):
    m = np.zeros((4, 4))
    for (i, j), s in pairs.items():
        m[i, j] = s
        m[j, i] = -s
    return m


# strain_k = 2 q^T B_k q' equals 2 vec(conj(q) q')_k
B1 = _skew_form({(0, 1): 1.0, (2, 3): -1.0})
B2 = _skew_form({(0, 2): 1.0, (1, 3): 1.0})
B3 = _skew_form({(0, 3): 1.0, (1, 2): -1.0})
B_MATRICES = np.stack([B1, B2, B3])
