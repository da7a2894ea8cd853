"""perfseer-b200: the B200-native measured-kernel and calibration path of
Stevens & Kloeckner (arXiv 1904.09538) behind the reference's
Executor / fit_model / predict interfaces. See DESIGN.md."""
from ._abi import KernelDesc, PsError, desc_from_id, kernel_io, lib  # noqa: F401

__all__ = ["KernelDesc", "PsError", "desc_from_id", "kernel_io", "lib"]
