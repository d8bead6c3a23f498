"""Import the upstream reference package from a throw-away copy.

Used ONLY by ``make_golden.py`` in the build container (the reference tree is
absent on GPU boxes).  Importing in place would write numba caches and
``__pycache__`` into the read-only reference mount (SURVEY.md §8c caveat), so
the package is copied to a temp dir first and numba's cache is redirected.
"""

from __future__ import annotations

import importlib
import os
import shutil
import sys
import tempfile

REF_SRC = "/root/reference/pkg/src/mdcontour"


def load_reference():
    if not os.path.isdir(REF_SRC):
        raise RuntimeError("reference tree not present (golden generation runs in the build container only)")
    tmp = tempfile.mkdtemp(prefix="mdc_ref_")
    shutil.copytree(REF_SRC, os.path.join(tmp, "mdcontour"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tmp, "numba_cache"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, tmp)
    mods = {}
    for name in ("dataset", "projection", "mesh", "bhtree", "layout", "field", "render", "_kernels", "cli"):
        mods[name] = importlib.import_module(f"mdcontour.{name}")
    return mods
