"""B200-native HydraServe cold-start path (arXiv 2502.15524): C-ABI library libhs.so
(include/hs.h) with tcgen05/TMA GEMMs and hand-written sm_100a kernels, and its thin ctypes
binding ``paper_2502_15524_b200.hs``.  See DESIGN.md."""
from . import hs  # noqa: F401
from .hs import Group, HostImage, DistComm, plan_stages, image_layout  # noqa: F401
