"""Parameter set of the DIS flow path — field-for-field the reference's
``DisParams`` / ``VarParams`` (reference pkg/src/disflow/core.py:197-319),
with the same defaults, presets, validation messages and exception type.

One documented extension: ``VarParams.outer_iters_fixed``.  The reference
runs ``outer_iters(s) = s + 1`` fixed-point iterations at scale ``s``
(core.py:212-213); the BASELINE configs ask for "1 outer / 5 inner", which the
reference can only express by subclassing ``VarParams``.  Setting
``outer_iters_fixed=k`` (k >= 1) makes ``outer_iters(s) == k`` here, and the
oracle/goldens apply the identical override on the reference side.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field, replace


class ParameterError(ValueError):
    """Invalid solver parameter or parameter combination (core.py:25-26)."""


def coarsest_scale_for(width: float, patch_size: int, motion_fraction: float,
                       downscale: int = 2) -> int:
    """core.py:131-147: smallest integer >= log_downscale(2*width /
    (motion_fraction*patch_size)), clamped at 0."""
    if width <= 0 or patch_size <= 0 or motion_fraction <= 0:
        raise ParameterError("width, patch_size, and motion_fraction must be > 0")
    arg = 2.0 * width / (motion_fraction * patch_size)
    if arg <= 1.0:
        return 0
    if downscale == 2:
        value = math.log2(arg)
    else:
        value = math.log(arg) / math.log(downscale)
    return max(0, math.ceil(value - 1e-9))


@dataclass(frozen=True)
class VarParams:
    """Variational refinement weights/iterations (core.py:197-223)."""

    intensity_weight: float = 5.0
    gradient_weight: float = 10.0
    smoothness_weight: float = 10.0
    inner_sor_iters: int = 5
    penalizer_eps: float = 0.001
    sor_omega: float = 1.6
    outer_iters_fixed: int | None = None  # extension (module docstring)

    def outer_iters(self, scale_index: int) -> int:
        if self.outer_iters_fixed is not None:
            return int(self.outer_iters_fixed)
        return scale_index + 1

    def validate(self) -> None:
        if self.intensity_weight < 0 or self.gradient_weight < 0 or self.smoothness_weight < 0:
            raise ParameterError("variational weights must be >= 0")
        if self.inner_sor_iters < 1:
            raise ParameterError("inner_sor_iters must be >= 1")
        if self.penalizer_eps <= 0:
            raise ParameterError("penalizer_eps must be > 0")
        if not 0.0 < self.sor_omega < 2.0:
            raise ParameterError("sor_omega must lie in (0, 2)")
        if self.outer_iters_fixed is not None and self.outer_iters_fixed < 1:
            raise ParameterError("outer_iters_fixed must be >= 1")


# operating points: (finest_scale, iterations, patch_size, overlap, refined)
# core.py:227-232
_PRESETS = {
    1: (3, 16, 8, 0.30, False),
    2: (3, 12, 8, 0.40, True),
    3: (1, 16, 12, 0.75, True),
    4: (0, 256, 12, 0.75, True),
}

RESIDUAL_NORMS = ("l2", "l1", "huber")
NORM_CODES = {"l2": 0, "l1": 1, "huber": 2}  # inverse_search.py:20


@dataclass(frozen=True)
class DisParams:
    """Full parameter set of the pipeline (core.py:237-319)."""

    patch_size: int = 8
    overlap: float = 0.40
    iterations: int = 12
    finest_scale: int = 3
    coarsest_scale: int = 5
    downscale: int = 2
    use_mean_normalization: bool = True
    use_densification: bool = True
    residual_norm: str = "l2"
    huber_b: float = 1.0
    variational: VarParams | None = field(default_factory=VarParams)
    mode: str = "flow"
    bidirectional: bool = False

    @classmethod
    def preset(cls, number: int, *, width: int | None = None,
               coarsest_scale: int | None = None, stereo: bool = False) -> "DisParams":
        """core.py:259-294."""
        if number not in _PRESETS:
            raise ParameterError(f"preset must be 1..4, got {number}")
        finest, iters, ps, ov, refined = _PRESETS[number]
        if stereo:
            iters //= 2
        if coarsest_scale is None:
            if width is not None:
                coarsest_scale = coarsest_scale_for(width, ps, 8.0)
            else:
                coarsest_scale = 5
        coarsest_scale = max(coarsest_scale, finest)
        return cls(
            patch_size=ps, overlap=ov, iterations=iters, finest_scale=finest,
            coarsest_scale=coarsest_scale,
            variational=VarParams() if refined else None,
            mode="stereo" if stereo else "flow",
        )

    def validate(self) -> None:
        """core.py:296-316."""
        if self.patch_size < 2:
            raise ParameterError("patch_size must be >= 2")
        if not 0.0 <= self.overlap < 1.0:
            raise ParameterError("overlap must lie in [0, 1)")
        if self.iterations < 1:
            raise ParameterError("iterations must be >= 1")
        if self.finest_scale < 0 or self.coarsest_scale < self.finest_scale:
            raise ParameterError("need 0 <= finest_scale <= coarsest_scale")
        if self.downscale < 2 or int(self.downscale) != self.downscale:
            raise ParameterError("downscale must be an integer >= 2")
        if self.residual_norm not in RESIDUAL_NORMS:
            raise ParameterError(f"residual_norm must be one of {RESIDUAL_NORMS}")
        if self.residual_norm == "huber" and self.huber_b <= 0:
            raise ParameterError("huber_b must be > 0")
        if self.mode not in ("flow", "stereo"):
            raise ParameterError("mode must be 'flow' or 'stereo'")
        if self.mode == "stereo" and self.bidirectional:
            raise ParameterError("bidirectional matching is not defined for stereo mode")
        if self.variational is not None:
            self.variational.validate()

    def without_variational(self) -> "DisParams":
        return replace(self, variational=None)


class DisParamsC(ctypes.Structure):
    """ctypes mirror of ``dis_params_t`` (include/dis_b200.h)."""

    _fields_ = [
        ("patch_size", ctypes.c_int32),
        ("iterations", ctypes.c_int32),
        ("finest_scale", ctypes.c_int32),
        ("coarsest_scale", ctypes.c_int32),
        ("downscale", ctypes.c_int32),
        ("use_mean_normalization", ctypes.c_int32),
        ("use_densification", ctypes.c_int32),
        ("residual_norm", ctypes.c_int32),
        ("overlap", ctypes.c_double),
        ("huber_b", ctypes.c_double),
        ("variational", ctypes.c_int32),
        ("var_inner_sor_iters", ctypes.c_int32),
        ("var_intensity_weight", ctypes.c_double),
        ("var_gradient_weight", ctypes.c_double),
        ("var_smoothness_weight", ctypes.c_double),
        ("var_penalizer_eps", ctypes.c_double),
        ("var_sor_omega", ctypes.c_double),
        ("outer_iters_fixed", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("bidirectional", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


def to_c(p: DisParams) -> DisParamsC:
    """Pack a DisParams into the C ABI struct."""
    c = DisParamsC()
    c.patch_size = int(p.patch_size)
    c.iterations = int(p.iterations)
    c.finest_scale = int(p.finest_scale)
    c.coarsest_scale = int(p.coarsest_scale)
    c.downscale = int(p.downscale)
    c.use_mean_normalization = int(bool(p.use_mean_normalization))
    c.use_densification = int(bool(p.use_densification))
    c.residual_norm = NORM_CODES.get(p.residual_norm, -1)
    c.overlap = float(p.overlap)
    c.huber_b = float(p.huber_b)
    vp = p.variational
    c.variational = 0 if vp is None else 1
    vp = vp if vp is not None else VarParams()
    c.var_inner_sor_iters = int(vp.inner_sor_iters)
    c.var_intensity_weight = float(vp.intensity_weight)
    c.var_gradient_weight = float(vp.gradient_weight)
    c.var_smoothness_weight = float(vp.smoothness_weight)
    c.var_penalizer_eps = float(vp.penalizer_eps)
    c.var_sor_omega = float(vp.sor_omega)
    c.outer_iters_fixed = 0 if vp.outer_iters_fixed is None else int(vp.outer_iters_fixed)
    c.mode = 0 if p.mode == "flow" else 1
    c.bidirectional = int(bool(p.bidirectional))
    c.reserved = 0
    return c
