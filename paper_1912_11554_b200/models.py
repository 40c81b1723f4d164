"""Target densities, executed on the device.

Reference: turnstile/models.py.  ``TargetModel`` keeps the reference's
fields (name, dim, potential, gradient, params) so code written against the
reference plugin API still reads the same.  Built-in constructors return
models whose ``potential``/``gradient`` callables evaluate on the GPU through
``ts_potential_grad`` and which carry a ``device_spec`` describing the
device-resident data (the reference hides X and y in closures,
models.py:107-118; here they are uploaded once and re-tiled in HBM).

A ``TargetModel`` built from arbitrary Python callables has no device
counterpart: the samplers reject it with ``ValueError`` (there is no CPU
fallback, BASELINE.json north star).
"""

from __future__ import annotations

import csv
import json
import warnings
from dataclasses import dataclass, field
from pathlib import Path
from typing import Callable, Optional

import numpy as np

from . import _lib

PRECISIONS = ("fp64", "fp32", "tf32", "fp64x")


class DeviceSpec:
    """Device description of a built-in model; owns per-GPU ts_model handles."""

    def __init__(self, kind: int, dim: int, params=None, x=None, y=None, precision: str = "fp64"):
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}")
        self.kind = kind
        self.dim = dim
        self.params = None if params is None else np.ascontiguousarray(params, dtype=np.float64)
        self.x = x  # fp32 (fp64 for "fp64x") (N, p) C-contiguous, logistic only
        self.y = y  # uint8 (N,)
        self.precision = precision
        self._handles: dict = {}
        self._grid = 0
        self.row_shard = None  # (rank, world) once joined by rowshard.connect
        self.reparam = None  # dense_gaussian with a dense mass: L (q = L x)

    def handle(self, device=None):
        """ts_model* for the given CUDA device (created on first use)."""
        torch = _lib.torch_cuda()
        dev = _lib.cuda_device(torch, device)
        key = dev.index
        h = self._handles.get(key)
        if h is not None:
            return h
        lib = _lib.load_library()
        out = _lib._P()
        with torch.cuda.device(dev):
            xd = yd = None
            n_rows = n_feat = 0
            if self.kind == _lib.TS_LOGISTIC:
                xd = torch.from_numpy(self.x).to(dev)
                yd = torch.from_numpy(self.y).to(dev)
                n_rows, n_feat = self.x.shape
            params = self.params
            pp = params.ctypes.data if params is not None else 0
            npar = 0 if params is None else params.size
            prec = {"fp64": _lib.TS_PREC_FP64, "fp32": _lib.TS_PREC_FP32, "tf32": _lib.TS_PREC_TF32,
                    "fp64x": _lib.TS_PREC_FP64X}[self.precision]
            _lib.check(lib.ts_model_create(self.kind, self.dim, pp, npar, _lib.ptr(xd), _lib.ptr(yd), n_rows, n_feat, prec,
                                           ctypes_byref(out)))
            if self._grid:
                _lib.check(lib.ts_model_set_grid(out, self._grid))
            torch.cuda.synchronize(dev)
        self._handles[key] = out
        return out

    def set_grid(self, grid: int) -> None:
        """Cap the persistent grid size (testing / multi-tenant use)."""
        self._grid = int(grid)
        lib = _lib.load_library()
        for h in self._handles.values():
            _lib.check(lib.ts_model_set_grid(h, self._grid))

    def __del__(self):
        try:
            lib = _lib._lib
            if lib is not None:
                for h in self._handles.values():
                    lib.ts_model_destroy(h)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


def ctypes_byref(x):
    import ctypes

    return ctypes.byref(x)


def potential_and_gradient(spec: DeviceSpec, qs: np.ndarray, device=None) -> np.ndarray:
    """Fused U and gradient at each row of ``qs`` -> array (n, 1 + dim)."""
    torch = _lib.torch_cuda()
    qs = np.atleast_2d(np.asarray(qs, dtype=np.float64))
    if qs.shape[1] != spec.dim:
        raise ValueError(f"expected parameter vector of length {spec.dim}, got {qs.shape[1]}")
    h = spec.handle(device)
    dev = _lib.cuda_device(torch, device)
    qd = torch.from_numpy(np.ascontiguousarray(qs)).to(dev)
    out = torch.empty((qs.shape[0], spec.dim + 1), dtype=torch.float64, device=dev)
    lib = _lib.load_library()
    with torch.cuda.device(dev):
        _lib.check(lib.ts_potential_grad(h, _lib.ptr(qd), qs.shape[0], _lib.ptr(out), _lib.stream_ptr(torch)))
    res = out.cpu().numpy()
    _lib.check_spec(spec, h)
    return res


@dataclass(frozen=True)
class TargetModel:
    """A target distribution seen through its potential energy surface."""

    name: str
    dim: int
    potential: Callable[[np.ndarray], float]
    gradient: Callable[[np.ndarray], np.ndarray]
    params: dict = field(default_factory=dict)
    device_spec: Optional[DeviceSpec] = field(default=None, compare=False, repr=False)

    def __post_init__(self):
        if self.dim < 1:
            raise ValueError("model dimension must be positive")

    def descriptor(self) -> dict:
        return {"model": self.name, "params": self.params}


def require_device(model: TargetModel) -> DeviceSpec:
    if model.device_spec is None:
        raise ValueError(
            f"model {model.name!r} has no device implementation; only the built-in models "
            f"{BUILTIN_MODELS} run on the B200 path (no CPU fallback)"
        )
    return model.device_spec


def _device_model(name: str, spec: DeviceSpec, params: dict) -> TargetModel:
    dim = spec.dim

    def potential(q: np.ndarray) -> float:
        return float(potential_and_gradient(spec, np.asarray(q, dtype=np.float64).reshape(1, -1))[0, 0])

    def gradient(q: np.ndarray) -> np.ndarray:
        return potential_and_gradient(spec, np.asarray(q, dtype=np.float64).reshape(1, -1))[0, 1:].copy()

    return TargetModel(name, dim, potential, gradient, params, spec)


@dataclass(frozen=True)
class LogisticRegressionData:
    """Covariates and binary labels (models.py:43-64).

    Kept in the device's storage types: X as float32 when every value is
    exactly representable in fp32 (the synthetic benchmark data are), else as
    float64 - never silently rounded (the reference keeps fp64,
    models.py:51-60); y as uint8.
    """

    x: np.ndarray
    y: np.ndarray

    def __post_init__(self):
        x = np.atleast_2d(np.asarray(self.x))
        y = np.asarray(self.y).ravel()
        if x.shape[0] != y.shape[0]:
            raise ValueError("covariate rows and labels disagree in length")
        if x.dtype == np.float32:
            xs = np.ascontiguousarray(x)
        else:
            x64 = np.ascontiguousarray(x, dtype=np.float64)
            x32 = x64.astype(np.float32)
            xs = x32 if np.array_equal(x32.astype(np.float64), x64) else x64
        if not np.isfinite(xs).all() or (y.dtype.kind == "f" and not np.isfinite(y).all()):
            raise ValueError("logistic data must be free of NaN/Inf")
        y8 = y.astype(np.uint8)
        if not np.array_equal(y8, y) or (y8 > 1).any():
            raise ValueError("labels must be 0 or 1")
        object.__setattr__(self, "x", xs)
        object.__setattr__(self, "y", np.ascontiguousarray(y8))

    @property
    def fp32_exact(self) -> bool:
        return self.x.dtype == np.float32

    @property
    def num_features(self) -> int:
        return self.x.shape[1]


def std_normal_model(dim: int) -> TargetModel:
    if dim < 1:
        raise ValueError("dim must be >= 1")
    return _device_model("std_normal", DeviceSpec(_lib.TS_STD_NORMAL, dim), {"dim": dim})


def gaussian_model(cov_diag) -> TargetModel:
    var = np.asarray(cov_diag, dtype=np.float64).ravel()
    if var.size < 1:
        raise ValueError("cov_diag must be non-empty")
    if not (np.isfinite(var).all() and (var > 0).all()):
        raise ValueError("variances must be positive and finite")
    inv_var = np.ascontiguousarray(1.0 / var)
    return _device_model("gaussian", DeviceSpec(_lib.TS_GAUSSIAN, var.size, params=inv_var), {"cov_diag": var.tolist()})


def logistic_regression_model(data: LogisticRegressionData, precision: str = "fp64") -> TargetModel:
    """Bayesian logistic regression with unit-normal priors (models.py:101-126).

    ``precision`` selects the arithmetic of the fused data pass:
    ``"fp64"`` (parity mode, differs from the reference only in summation
    order), ``"fp32"`` (per-row math in float, accumulation in double) or
    ``"tf32"`` (many chains sharing X: each batched step streams X once for
    every chain with an outstanding gradient request and evaluates eta = X
    theta and X^T r on the tcgen05 tensor cores in 3xTF32 split precision,
    csrc/ts_k_logistic_many.cu; num_features <= 62).  fp32/fp64 runs of C
    chains launch the single-chain persistent pass C times; tf32 runs all
    chains in one launch.  ``"fp64x"`` streams X stored in fp64 (twice the
    bytes, no conversions); ``"fp64"`` on data that are not fp32-exact uses
    it automatically, the fp32 and tf32 policies round such data to fp32
    (within their stated tolerances) with a RuntimeWarning.
    """
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}")
    x, y8 = data.x, data.y
    if x.dtype == np.float64 and precision == "fp64":
        precision = "fp64x"
    elif x.dtype == np.float64 and precision in ("fp32", "tf32"):
        warnings.warn(f"logistic data are not fp32-exact; the {precision} policy rounds X to fp32", RuntimeWarning)
        x = x.astype(np.float32)
    elif precision == "fp64x":
        x = x.astype(np.float64)
    dim = data.num_features + 1
    spec = DeviceSpec(_lib.TS_LOGISTIC, dim, x=np.ascontiguousarray(x), y=y8, precision=precision)
    return _device_model(
        "logistic_regression",
        spec,
        {"num_data": int(x.shape[0]), "num_features": int(x.shape[1])},
    )


def funnel_model(dim: int = 10) -> TargetModel:
    if dim < 2:
        raise ValueError("funnel needs the scale coordinate plus at least one other")
    return _device_model("funnel", DeviceSpec(_lib.TS_FUNNEL, dim), {"dim": dim})


EIGHT_SCHOOLS_Y = (28.0, 8.0, -3.0, 7.0, -1.0, 1.0, 18.0, 12.0)
EIGHT_SCHOOLS_SIGMA = (15.0, 10.0, 16.0, 11.0, 9.0, 11.0, 10.0, 18.0)


def eight_schools_model(y=EIGHT_SCHOOLS_Y, sigma=EIGHT_SCHOOLS_SIGMA) -> TargetModel:
    """Non-centred eight schools: q = (mu, log tau, theta~_1..J).

    U = mu^2/50 + log1p((tau/5)^2) - log tau + sum_j [th_j^2/2 + ((y_j - mu - tau th_j)/sigma_j)^2/2]
    (mu ~ N(0, 5^2), tau ~ HalfCauchy(5), theta~ ~ N(0, 1)).
    """
    y = np.asarray(y, dtype=np.float64).ravel()
    s = np.asarray(sigma, dtype=np.float64).ravel()
    if y.size != s.size or y.size < 1:
        raise ValueError("y and sigma must be non-empty and of equal length")
    if not (np.isfinite(s).all() and (s > 0).all()):
        raise ValueError("sigma must be positive and finite")
    spec = DeviceSpec(_lib.TS_EIGHT_SCHOOLS, y.size + 2, params=np.concatenate([y, s]))
    return _device_model("eight_schools", spec, {"y": y.tolist(), "sigma": s.tolist()})


def dense_gaussian_model(precision_matrix, inv_mass=None, precision: str = "tf32") -> TargetModel:
    """Correlated Gaussian U(q) = q'Pq/2 on the many-chain lockstep path
    (no reference built-in, oracle twin in oracle/).

    Every leapfrog of every chain needs g = P q: the device batches all
    chains into one GEMM per lockstep step on the tcgen05 tensor cores
    (``precision="tf32"``, stated tolerance) or on the SIMT fp64 pipe
    (``"fp64"``, the parity policy).

    ``inv_mass`` (optional, dense SPD M^-1): NUTS with mass matrix M on U is
    run as identity-mass NUTS on x = L^-1 q, M^-1 = L L^T -- the same kinetic
    energy (r'M^-1 r = r_x'r_x), U-turn criterion and leapfrog map -- so the
    device model is U(x) = x'Ax/2 with A = L^T P L, and samples come back as
    q = L x.  The reference itself is diagonal-mass only (integrator.py:21-31).
    """
    P = np.asarray(precision_matrix, dtype=np.float64)
    if P.ndim != 2 or P.shape[0] != P.shape[1] or P.shape[0] < 1:
        raise ValueError("precision_matrix must be a non-empty square matrix")
    if not np.isfinite(P).all():
        raise ValueError("precision_matrix must be finite")
    D = P.shape[0]
    L = None
    if inv_mass is not None:
        Minv = np.asarray(inv_mass, dtype=np.float64)
        if Minv.shape != P.shape:
            raise ValueError("inv_mass must have the shape of precision_matrix")
        try:
            L = np.linalg.cholesky(Minv)
        except np.linalg.LinAlgError as e:
            raise ValueError("inv_mass must be symmetric positive definite") from e
        A = L.T @ P @ L
    else:
        A = P
    spec = DeviceSpec(_lib.TS_DENSE_GAUSS, D, params=np.ascontiguousarray(A).ravel(), precision=precision)
    spec.reparam = L
    params = {"dim": D, "dense_mass": L is not None}
    if L is None:
        return _device_model("dense_gaussian", spec, params)

    # user-facing potential / gradient in q coordinates (q = L x)
    def potential(q):
        x = np.linalg.solve(L, np.asarray(q, dtype=np.float64))
        return float(potential_and_gradient(spec, x.reshape(1, -1))[0, 0])

    def gradient(q):
        x = np.linalg.solve(L, np.asarray(q, dtype=np.float64))
        return np.linalg.solve(L.T, potential_and_gradient(spec, x.reshape(1, -1))[0, 1:])

    return TargetModel("dense_gaussian", D, potential, gradient, params, spec)


def fd_gradient(model: TargetModel, q: np.ndarray, h: float = 1e-5) -> np.ndarray:
    """Central-difference gradient oracle (models.py:147-160)."""
    if h <= 0:
        raise ValueError("step h must be positive")
    q = np.asarray(q, dtype=np.float64)
    out = np.empty_like(q)
    for i in range(q.size):
        bumped = q.copy()
        bumped[i] = q[i] + h
        up = model.potential(bumped)
        bumped[i] = q[i] - h
        down = model.potential(bumped)
        out[i] = (up - down) / (2.0 * h)
    return out


def load_logistic_csv(path) -> LogisticRegressionData:
    rows = []
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader, None)
        if header is None:
            raise ValueError(f"{path}: empty CSV")
        for row in reader:
            if row:
                rows.append([float(v) for v in row])
    if not rows:
        raise ValueError(f"{path}: no data rows")
    mat = np.asarray(rows, dtype=np.float64)
    return LogisticRegressionData(mat[:, :-1], mat[:, -1])


def model_from_descriptor(descriptor, base_dir=None) -> TargetModel:
    """Build a model from a JSON descriptor (models.py:180-215)."""
    if isinstance(descriptor, (str, Path)):
        p = Path(descriptor)
        if p.exists():
            desc = json.loads(p.read_text())
            base_dir = p.parent if base_dir is None else base_dir
        else:
            desc = json.loads(str(descriptor))
    else:
        desc = dict(descriptor)
    name = desc.get("model")
    params = dict(desc.get("params") or {})
    if name == "std_normal":
        return std_normal_model(int(params.get("dim", 1)))
    if name == "gaussian":
        if "cov_diag" not in params:
            raise ValueError("gaussian descriptor needs params.cov_diag")
        return gaussian_model(params["cov_diag"])
    if name == "funnel":
        return funnel_model(int(params.get("dim", 10)))
    if name == "eight_schools":
        return eight_schools_model(params.get("y", EIGHT_SCHOOLS_Y), params.get("sigma", EIGHT_SCHOOLS_SIGMA))
    if name == "logistic_regression":
        data_path = desc.get("data_path")
        if data_path is None:
            raise ValueError("logistic_regression descriptor needs data_path")
        data_path = Path(data_path)
        if not data_path.is_absolute() and base_dir is not None:
            data_path = Path(base_dir) / data_path
        return logistic_regression_model(load_logistic_csv(data_path), precision=params.get("precision", "fp64"))
    raise ValueError(f"unknown model name: {name!r}")


BUILTIN_MODELS = ("std_normal", "gaussian", "logistic_regression", "funnel", "eight_schools", "dense_gaussian")
