"""Interpreter-start hook for the reference-suite runs (test infrastructure).

Only active when LCPSEARCH_GPU_SHIM is set: installs the GPU shim into the
reference ``lcpsearch`` (see lcpsearch_gpu_shim.py).  The system
sitecustomize this file shadows on PYTHONPATH is executed first.
"""

import os
import sys

_here = os.path.dirname(os.path.abspath(__file__))
for _p in sys.path:
    _f = os.path.join(_p, "sitecustomize.py")
    if _p and os.path.abspath(_p) != _here and os.path.isfile(_f):
        with open(_f) as _fh:
            exec(compile(_fh.read(), _f, "exec"), {"__name__": "sitecustomize", "__file__": _f})
        break

if os.environ.get("LCPSEARCH_GPU_SHIM"):
    import lcpsearch_gpu_shim

    lcpsearch_gpu_shim.install()
