"""Device-resident estimator plan (qt_plan_* of include/qtree_cuda.h).

PyTorch is used only for device memory, streams and torch.distributed; every
count is produced by libqtree_cuda.so's kernels. One Plan per GPU: the grids
are staged once, then `count()` enqueues the fused path kernel for any unit
window on the current torch stream, and `finalize()` derives visits + pi.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L
from .qtree import EstimatorKind, _check, _GridPack, layout


class Plan:
    def __init__(self, chain, grids, device: int = 0):
        self.chain = chain
        self.device = int(device)
        self._gp = _GridPack(chain, grids)
        self.sizes = self._gp.sizes
        self.n_visits, self.n_joint = layout(self.sizes)
        h = C.c_void_p()
        ch = chain.c()
        _check(L.lib().qt_plan_create(C.byref(ch), C.byref(self._gp.s), self.device, C.byref(h)),
               "plan_create")
        self._h = h
        self.launches = 0

    def close(self):
        if self._h:
            L.lib().qt_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def zeros_joint(self) -> torch.Tensor:
        return torch.zeros(self.n_joint, dtype=torch.int64, device=f"cuda:{self.device}")

    def count(self, estimator, engine, seed, first, count, total, joint: torch.Tensor,
              normals: torch.Tensor | None = None, stream=None) -> int:
        """Enqueue units [first, first+count) of `total` into `joint` (ADDED)."""
        assert joint.is_cuda and joint.dtype == torch.int64 and joint.numel() == self.n_joint
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        n = C.c_int32(0)
        _check(L.lib().qt_plan_count(self._h, int(estimator), int(engine), int(seed), int(first),
                                     int(count), int(total),
                                     C.c_void_p(normals.data_ptr()) if normals is not None else None,
                                     C.c_void_p(joint.data_ptr()), C.c_void_p(st.cuda_stream),
                                     C.byref(n)), "plan_count")
        self.launches += n.value
        return n.value

    def finalize(self, estimator, samples, joint: torch.Tensor, visits: torch.Tensor,
                 pi: torch.Tensor, stream=None) -> int:
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        n = C.c_int32(0)
        _check(L.lib().qt_plan_finalize(self._h, int(estimator), int(samples),
                                        C.c_void_p(joint.data_ptr()), C.c_void_p(visits.data_ptr()),
                                        C.c_void_p(pi.data_ptr()), C.c_void_p(st.cuda_stream),
                                        C.byref(n)), "plan_finalize")
        self.launches += n.value
        return n.value


    def save_tree(self, path, samples: int, joint: torch.Tensor, visits: torch.Tensor,
                  pi: torch.Tensor, x0=None) -> None:
        """Write the device-resident tree as QTRE v1 (quant_tree.hpp:138-163) straight
        from HBM through pinned staging buffers (no host copy of the counts / pi)."""
        import numpy as np
        torch.cuda.synchronize(self.device)
        dim = self.chain.dim()
        x0 = np.zeros(dim) if x0 is None else np.asarray(x0, np.float64)
        pts = np.ascontiguousarray(np.concatenate([x0, self._gp.points]), np.float64)
        sizes = np.ascontiguousarray(self.sizes, np.uint64)
        _check(L.lib().qt_save_tree(str(path).encode(), len(sizes) - 1, dim,
                                    sizes.ctypes.data_as(C.POINTER(C.c_uint64)),
                                    pts.ctypes.data_as(C.POINTER(C.c_double)), int(samples),
                                    C.c_void_p(visits.data_ptr()), C.c_void_p(joint.data_ptr()),
                                    C.c_void_p(pi.data_ptr()), 1), "save_tree")

    def fast_stats(self) -> dict:
        """Fast 1-D path evidence of this plan (synchronises its device)."""
        out = (C.c_uint64 * 3)()
        _check(L.lib().qt_plan_fast_stats(self._h, out), "plan_fast_stats")
        return {"fast_paths": int(out[0]), "replayed": int(out[1]), "inline_replayed": int(out[2])}


def units_total(estimator, chain, samples: int) -> int:
    return samples * chain.layers() if int(estimator) == EstimatorKind.AlgIII else samples
