"""Training-loop hook: keep a weight inside a bi-level ball after every step.

The reference's training program projects its weight after every gradient
step so each feature group satisfies the bi-level (1, q) constraint
(``project_features``, proj/src/train.cpp:26-30, called at :181,199; config 5 of
BASELINE.json is that per-step projection at scale).  There the weight is
W (features x classes) and the projection runs on a host transpose.  On the
GPU the projection runs in place on the parameter's storage:

* a ``torch.nn.Linear`` weight (out_features x in_features) already has the
  input features as columns -- the fibers of ``mp_bilevel_project`` -- so the
  hook projects it with no copy and can sit inside a captured training-step
  graph (``feature_dim=1``, the default);
* a features-as-rows weight (the reference's W layout, ``feature_dim=0``) is
  projected through one transposed copy each way.
"""
from __future__ import annotations

from ._capi import MpShapeError, norm_code
from . import BilevelProjector


class FeatureProjector:
    """``hook()`` projects ``weight`` in place onto {W : sum_f ||W_f||_q <= eta}
    (outer l1 over the feature groups f, inner q-norm within a group) without
    a host sync; ``zero_features()`` reads the number of zeroed feature groups
    of the last call (that read syncs)."""

    def __init__(self, weight, eta: float, q="inf", feature_dim: int = 1, flags: int = 0):
        import torch
        if weight.dim() != 2:
            raise MpShapeError("FeatureProjector needs a 2-D weight")
        if feature_dim not in (0, 1):
            raise MpShapeError("feature_dim must be 0 (rows) or 1 (columns)")
        if weight.dtype not in (torch.float32, torch.float64) or not weight.is_cuda:
            raise MpShapeError("FeatureProjector needs a float32/float64 CUDA weight")
        self.weight = weight
        self.eta = float(eta)
        self.feature_dim = feature_dim
        n, m = (weight.shape[0], weight.shape[1]) if feature_dim == 1 else (weight.shape[1], weight.shape[0])
        if feature_dim == 1 and not weight.is_contiguous():
            raise MpShapeError("feature_dim=1 needs a contiguous weight (columns are the feature groups)")
        self.proj = BilevelProjector(n, m, weight.dtype, "1", norm_code(q), weight.device, flags)
        self.scratch = None if feature_dim == 1 else torch.empty((n, m), dtype=weight.dtype, device=weight.device)

    def __call__(self, stream=None):
        import torch
        with torch.no_grad():
            if self.feature_dim == 1:
                self.proj(self.weight.data, self.weight.data, self.eta, stream=stream)
            else:
                self.scratch.copy_(self.weight.data.t())
                self.proj(self.scratch, self.scratch, self.eta, stream=stream)
                self.weight.data.copy_(self.scratch.t())
        return self

    def zero_features(self) -> int:
        return int(self.proj.info().zero_columns)

    @property
    def budgets(self):
        """Per-feature budgets u_f of the last projection (device tensor)."""
        return self.proj.budgets
