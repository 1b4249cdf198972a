"""ORACLE -- test infrastructure, never the product path.

A CPU restatement (numpy) of the reference's `ml(infer)` region path, used
only by tests/, `__graft_entry__.smoke()` and bench.py's cpu_baseline /
`--impl reference` leg as the checker.  Each function cites the reference
code it restates.  It is pinned against golden vectors produced by the
reference itself (tests/golden/make_golden.py imports /root/reference in the
build container; tests/test_oracle.py checks this module against them).

Arrays are passed as (flat ndarray, shape, element strides), the reference's
ArrayBuffer triple (bridge.py:76-126).

The gather here is written from the functor semantics directly (the k-th LHS
symbol sweeps the k-th target slice; a symbolic RHS dim is the symbol's value
plus an offset or offset range; a constant RHS dim is an absolute index),
independently of the bridge's stride machinery -- the same role
`gather_oracle` plays in the reference tests (tests/helpers.py:37-51), but
vectorised so it finishes full-size configs.
"""

from __future__ import annotations

import numpy as np

__all__ = ["slice_index_grid", "gather", "scatter", "infer", "region", "dense_relu_model",
           "init_mlp_f32"]


def _dim_values(dim, sym_axis, sweep_vals):
    """Index values of one RHS dim: shape (sweep..., count)."""
    if dim.symbol is None:
        if dim.stop is None:
            vals = np.array([dim.start.offset])
        else:
            vals = np.arange(dim.start.offset, dim.stop.offset, dim.step)
        return None, vals
    k = sym_axis[dim.symbol]
    if dim.stop is None:
        rel = np.array([dim.start.offset])
    else:
        rel = np.arange(dim.start.offset, dim.stop.offset, dim.step)
    return k, rel


def slice_index_grid(functor, target, shape, strides):
    """Flat element addresses of every (sweep point, feature) of the functor
    applied to the target: int64 array (sweep..., F), feature order = RHS
    declaration order, row-major within a slice (bridge.py:351-381).
    Raises IndexError on an out-of-bounds index (bridge.py:322-326)."""
    syms = functor.symbols
    sym_axis = {s: k for k, s in enumerate(syms)}
    sweep_vals = [np.arange(s.start, s.stop, s.step, dtype=np.int64) for s in target.slices]
    sweep_shape = tuple(len(v) for v in sweep_vals)
    n_sweep = len(sweep_shape)
    cols = []
    for s in functor.rhs:
        if len(s.dims) != len(shape):
            raise IndexError("rank mismatch")
        per_dim = []
        for d_i, dim in enumerate(s.dims):
            k, vals = _dim_values(dim, sym_axis, sweep_vals)
            if k is None:
                idx = np.broadcast_to(vals.astype(np.int64), (1,) * n_sweep + (len(vals),))
            else:
                sv = sweep_vals[k].reshape([-1 if a == k else 1 for a in range(n_sweep)] + [1])
                idx = sv + vals.astype(np.int64).reshape((1,) * n_sweep + (-1,))
            if idx.size and (idx.min() < 0 or idx.max() >= shape[d_i]):
                raise IndexError(f"index out of bounds on dim {d_i}")
            per_dim.append(idx)
        # combine dims: feature axes row-major in dim order
        addr = np.zeros(sweep_shape + (1,), dtype=np.int64)
        for d_i, idx in enumerate(per_dim):
            full = np.broadcast_to(idx, sweep_shape + (idx.shape[-1],))
            addr = (addr[..., :, None] + full[..., None, :] * strides[d_i]).reshape(sweep_shape + (-1,))
        cols.append(addr)
    return np.concatenate(cols, axis=-1)


def gather(functor, target, data, shape, strides):
    """concretize_to (bridge.py:388-395) -> (sweep..., feature_sizes...)."""
    addr = slice_index_grid(functor, target, shape, strides)
    out = data[addr]
    return out.reshape(addr.shape[:-1] + tuple(functor.feature_sizes))


def scatter(functor, target, values, data, shape, strides):
    """scatter_from (bridge.py:407-454): point slices only, injective, cast to
    the array dtype; writes `data` in place."""
    for s in functor.rhs:
        for d in s.dims:
            if d.stop is not None:
                raise ValueError("non-injective: range slice")
    addr = slice_index_grid(functor, target, shape, strides)
    flat = addr.reshape(-1)
    if np.unique(flat).size != flat.size:
        raise ValueError("non-injective: duplicate destinations")
    n_sweep = len(target.slices)
    v = np.asarray(values).reshape(addr.shape[:n_sweep] + (-1,))
    data[addr] = v.astype(data.dtype, copy=False)


def infer(layers, x):
    """models.infer (models.py:197-224) with _matmul_rowwise (models.py:188-194):
    f32, per output: acc=0; acc = acc + x_f*w_f in feature order; + bias; act.
    layers: [(W [out,in] f32, b [out] f32, act)].  Returns (y f32, finite)."""
    y = np.ascontiguousarray(x, dtype=np.float32)
    with np.errstate(over="ignore", invalid="ignore"):
        for w, b, act in layers:
            w = np.asarray(w, np.float32)
            acc = np.zeros((y.shape[0], w.shape[0]), dtype=np.float32)
            for f in range(w.shape[1]):
                acc += y[:, f, None] * w[None, :, f]
            y = acc + np.asarray(b, np.float32)
            if act == "relu":
                y = np.maximum(y, np.float32(0.0))
            elif act == "tanh":
                y = np.tanh(y)
    return y, bool(np.isfinite(y).all())


def region(in_maps, out_maps, layers):
    """Runtime._run_surrogate (runtime.py:308-370): gather every in map
    (in+inout order), concat on F, infer, split columns over out maps
    (out+inout order), scatter.  maps: [(functor, target, data, shape, strides)].
    Returns (x [B,F], y [B,G], finite) and writes the out arrays."""
    xs = []
    for f, t, d, sh, st in in_maps:
        g = gather(f, t, d, sh, st)
        xs.append(g.reshape(-1, f.feature_count))
    x = xs[0] if len(xs) == 1 else np.concatenate(xs, axis=1)
    y, finite = infer(layers, x)
    if finite:
        col = 0
        for f, t, d, sh, st in out_maps:
            g = f.feature_count
            chunk = y[:, col:col + g]
            wide = chunk.astype(np.float64) if x.dtype == np.float64 else chunk
            scatter(f, t, wide, d, sh, st)
            col += g
    return x, y, finite


def init_mlp_f32(dims, activation="relu", seed=0, bias_seed=1, bias_std=0.1):
    """The frozen configs' weights: He init for relu,
    Glorot-style otherwise, drawn like smlrt_train.mlp.init_mlp
    (trainer/src/smlrt_train/mlp.py:94-103) from default_rng(seed) in layer
    order, cast to f32; biases replaced by N(0, bias_std) from default_rng(bias_seed)."""
    rng = np.random.default_rng(seed)
    ws = []
    for fi, fo in zip(dims, dims[1:]):
        scale = np.sqrt(2.0 / fi) if activation == "relu" else np.sqrt(1.0 / fi)
        ws.append(rng.normal(0.0, scale, size=(fo, fi)).astype(np.float32))
    brng = np.random.default_rng(bias_seed)
    bs = [brng.normal(0.0, bias_std, size=fo).astype(np.float32) for fo in dims[1:]]
    acts = [activation] * (len(dims) - 2) + ["identity"]
    return list(zip(ws, bs, acts))


def dense_relu_model(dims, seed=0):
    return init_mlp_f32(dims, "relu", seed)


def conv2d_patches(images, weights, bias, kernel, act):
    """conv2d (stride == kernel) as the reference expresses it: the patch
    functor [n, i, j, 0:k, 0:k] = ([n, i:i+k, j:j+k]) gathered by
    concretize_to (bridge.py:388-395) fed to a dense layer via infer
    (models.py:197-224).  images [N, C, H, W] -> [N, OC, H/k, W/k]."""
    n, c, h, w = images.shape
    k = kernel
    oh, ow = h // k, w // k
    patches = images.reshape(n, c, oh, k, ow, k).transpose(0, 2, 4, 1, 3, 5).reshape(n * oh * ow, c * k * k)
    y, _ = infer([(weights, bias, act)], patches)
    return y.reshape(n, oh, ow, -1).transpose(0, 3, 1, 2)


def maxpool2d(x, k):
    """k x k max pooling, NaN-propagating (np.max), [N, C, H, W]."""
    n, c, h, w = x.shape
    return x.reshape(n, c, h // k, k, w // k, k).max(axis=(3, 5))


def cnn_forward(layers, x, input_shape):
    """layers: [("conv2d", W, b, k, act) | ("maxpool2d", k) | ("dense", W, b, act)];
    x [N, C*H*W] -> (y [N, G], finite).  Flattening is (channel, row, col)."""
    h = np.asarray(x, dtype=np.float32).reshape((-1,) + tuple(input_shape))
    for L in layers:
        if L[0] == "conv2d":
            h = conv2d_patches(h, L[1], L[2], L[3], L[4])
        elif L[0] == "maxpool2d":
            h = maxpool2d(h, L[1])
        else:
            h, _ = infer([(L[1], L[2], L[3])], h.reshape(h.shape[0], -1))
    y = h.reshape(h.shape[0], -1)
    return y, bool(np.isfinite(y).all())
