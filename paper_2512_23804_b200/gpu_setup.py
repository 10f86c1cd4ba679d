"""GPU setup pipeline: coefficient fields and the
t-stacked operator values built on the device.

The host setup (problems.build_problem) assembles every A_t with SciPy
(reference fem.py:171-206) and then re-lays the values out for the device;
for config 3 that is 924 matrices (~4 s).  Here:

* lognormal gPC coefficient fields (reference random_field.py:130-151) come
  from `sgk_lognormal_fields` (one thread per (term, Gauss point));
* all stiffness slices and the mass matrix are assembled by `sgk_q1_assemble`
  straight into both device layouts of one `DevicePattern`
  (`DevicePattern.assemble_q1`);
* the host matrices the rest of the API expects (`bundle.stiffness`,
  `bundle.mass`: the lead factorisation, the oracle in tests) are views of one
  device-to-host copy of the values on the shared structure, and every
  operator built from them reuses the device pattern instead of re-uploading
  (`attached_pattern`).

The KL modes themselves stay on the host (one small eigenproblem).
"""

from __future__ import annotations

import math
import time
import weakref

import numpy as np
import scipy.sparse as sp
import torch

from . import _lib, fem
from .basis import build_triple_products, enumerate_multi_indices, level_partition
from .device import DevicePattern, device
from .random_field import CovarianceSpec, kl_expand

__all__ = ["attached_pattern", "build_problem_device", "lognormal_fields_device"]

# id(host matrix) -> (weak ref to the matrix, device pattern, slice index):
# host matrices that are views of a device-assembled pattern; entries go away
# with their matrices
_SLICES: dict[int, tuple[weakref.ref, DevicePattern, int]] = {}


def attached_pattern(mats) -> DevicePattern | None:
    """The device pattern whose slices 0..len(mats)-1 are exactly `mats`
    (same objects, in order), if they came from the device assembly."""
    pat = None
    for t, m in enumerate(mats):
        hit = _SLICES.get(id(m))
        if hit is None or hit[0]() is not m or hit[2] != t or (pat is not None and hit[1] is not pat):
            return None
        pat = hit[1]
    return pat


def lognormal_fields_device(modes, coeff_basis) -> torch.Tensor:
    """(n_terms, n_elements, 4) gPC coefficient fields of exp(g) on the device
    (reference random_field.py:130-151)."""
    if coeff_basis.m_xi != modes.m_xi:
        raise ValueError("coefficient basis and modes use different variable counts")
    mean = np.ascontiguousarray(modes.mean_field.values, np.float64)
    if np.any(mean <= 0):
        raise ValueError("lognormal mean field must be strictly positive")
    shape = mean.shape
    dev = device()
    mean_d = torch.as_tensor(mean.reshape(-1)).to(dev)
    g_d = torch.as_tensor(np.stack([f.values.reshape(-1) for f in modes.mode_fields])
                          if modes.m_xi else np.zeros((0, mean.size))).to(dev).contiguous()
    idx = torch.as_tensor(np.asarray(coeff_basis.as_array(), np.int32)).to(dev).contiguous()
    n_terms = idx.shape[0]
    out = torch.empty((n_terms,) + shape, dtype=torch.float64, device=dev)
    rc = _lib.lib().sgk_lognormal_fields(mean.size, modes.m_xi, n_terms, mean_d.data_ptr(),
                                         g_d.data_ptr() if modes.m_xi else None, idx.data_ptr(), out.data_ptr(),
                                         _lib.stream_ptr())
    _lib.check(rc, "sgk_lognormal_fields")
    return out


def build_problem_device(cfg, *, n: int | None = None, kl_method: str = "separable", beta: float | None = None):
    """problems.build_problem with the coefficient fields (lognormal) and all
    operator values built on the GPU.  Returns the same ProblemBundle; its
    host matrices are views of the device-assembled values and the device
    pattern is attached (no second upload).  bundle.extras["setup_seconds"]
    holds the timing split."""
    from dataclasses import replace

    from .problems import BASELINE_CONFIGS, ProblemBundle
    from .random_field import GpcCoefficientField, affine_coefficient

    spec = BASELINE_CONFIGS[cfg] if isinstance(cfg, int) else cfg
    if n is not None or beta is not None:
        spec = replace(spec, n=n if n is not None else spec.n, beta=beta if beta is not None else spec.beta)
    t0 = time.perf_counter()
    grid = fem.build_grid(spec.n, spec.lo, spec.hi)
    basis = enumerate_multi_indices(spec.m_xi, spec.p)
    partition = level_partition(basis)
    modes = kl_expand(CovarianceSpec(sigma_k=spec.sigma, ell1=spec.ell, ell2=spec.ell, mean=1.0), grid,
                      spec.m_xi, method=kl_method)
    if spec.coefficient == "affine":
        coeff_idx = enumerate_multi_indices(spec.m_xi, 1)
        gpc = affine_coefficient(modes, spec.family)
        fields = torch.as_tensor(np.stack([f.values for f in gpc.coeff_fields])).to(device())
    else:
        coeff_idx = enumerate_multi_indices(spec.m_xi, spec.coefficient_degree)
        fields = lognormal_fields_device(modes, coeff_idx)
        gpc = None
    triple = build_triple_products(basis, coeff_idx, spec.gamma, family=spec.family)
    t1 = time.perf_counter()
    pat = DevicePattern.assemble_q1(grid, fields, with_mass=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    data = pat.slice_data  # one device-to-host copy of all slices
    T = pat.n_slices - 1
    ip, ix = pat.indptr.astype(np.int32), pat.indices.astype(np.int32)
    mats = [sp.csr_matrix((data[t], ix, ip), shape=(pat.n_rows, pat.n_rows)) for t in range(T + 1)]
    for t, m in enumerate(mats):
        _SLICES[id(m)] = (weakref.ref(m), pat, t)
        weakref.finalize(m, _SLICES.pop, id(m), None)
    if gpc is None:
        host_fields = fields.cpu().numpy()
        gpc = GpcCoefficientField(coeff_fields=[fem.CoefficientField(values=v) for v in host_fields])
    t3 = time.perf_counter()
    bundle = ProblemBundle(spec, grid, basis, partition, triple, modes, gpc, mats[T], mats[:T])
    bundle.extras["setup_seconds"] = {"fields_kl_triples": t1 - t0, "device_assembly": t2 - t1,
                                      "host_views": t3 - t2, "total": t3 - t0}
    bundle.extras["device_pattern"] = pat
    return bundle
