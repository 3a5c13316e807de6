"""The reference package `sdmortar`, whose objects this drop-in consumes.

The drop-in accelerates `sdmortar.interface.run_method` for a caller who
already holds `sdmortar` objects, so `sdmortar` is a dependency of the host
side, like numpy. It is imported from the environment; when it is not
installed there, from the repo's own install location `baseline/_ref`
(`pip install --target baseline/_ref <sdmortar>`).
"""

import importlib
import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
_VENDORED = os.path.join(os.path.dirname(_HERE), "baseline", "_ref")

try:
    import sdmortar  # noqa: F401
except ImportError:
    if os.path.isdir(os.path.join(_VENDORED, "sdmortar")):
        sys.path.append(_VENDORED)
    import sdmortar  # noqa: F401  (ImportError here: sdmortar is required)

for _m in ("collocation", "config", "darcy", "errors", "geometry", "interface", "moments",
           "mortar", "output", "problem", "random_field", "stokes"):
    importlib.import_module(f"sdmortar.{_m}")
