"""Assemble an `altotensor` package whose hot-path modules are the drop-in.

SURVEY.md §7.2 item 8: run the reference's own test suite unchanged against
the device path.  The shim package is written into a scratch directory:

  altotensor/layout.py, format.py, mttkrp.py, cpd.py
      re-export paper_2102_10245_b200's modules (the B200 hot path), plus
      the reference's out-of-scope reporting names (storage_stats /
      StorageStats) taken from the unmodified reference;
  altotensor/__init__.py, coo.py, container.py, cli.py
      copied verbatim from the installed reference (baseline/_ref): the
      modules SURVEY §2 keeps out of scope; their relative imports
      (`from .format import ...`) bind to the drop-in modules above;
  _altoref/
      the whole unmodified reference package under another name, the source
      of the reporting names above.

Nothing here is copied into the repository: the reference files are read
from baseline/_ref at test time (git-ignored; it travels to the GPU box).
"""

from __future__ import annotations

import os
import shutil

HOT = {
    "layout": ("from _altoref.layout import StorageStats, storage_stats  # reporting (out of scope)\n"),
    "format": "",
    "mttkrp": "",
    "cpd": "",
}


def build_shim(dest: str, ref_pkg: str) -> str:
    """Write the shim into `dest`; `ref_pkg` is the installed reference's
    `altotensor` directory.  Returns `dest` (put it first on sys.path)."""
    shutil.copytree(ref_pkg, os.path.join(dest, "_altoref"), dirs_exist_ok=True,
                    ignore=shutil.ignore_patterns("__pycache__"))
    pkg = os.path.join(dest, "altotensor")
    os.makedirs(pkg, exist_ok=True)
    for name in ("__init__", "coo", "container", "cli"):
        shutil.copyfile(os.path.join(ref_pkg, f"{name}.py"), os.path.join(pkg, f"{name}.py"))
    for name, extra in HOT.items():
        src = (f'"""Drop-in: paper_2102_10245_b200.{name} (B200 hot path)."""\n'
               f"import sys as _sys\n"
               f"import paper_2102_10245_b200.{name} as _m\n"
               f"from paper_2102_10245_b200.{name} import *  # noqa: F401,F403\n"
               f"globals().update({{k: v for k, v in vars(_m).items() if not k.startswith('__')}})\n"
               f"{extra}")
        with open(os.path.join(pkg, f"{name}.py"), "w") as f:
            f.write(src)
    return dest
