"""Imports the reference implementation built by oracle/build_ref.py —
TEST INFRASTRUCTURE (bench.py reference arm, tests).

The pure-Python modules are extracted from oracle/_ref/dhgpart_ref.zip into a
fresh temporary directory next to the compiled kernel module, so the import
never depends on anything left over in /tmp from an earlier call.
"""
from __future__ import annotations

import shutil
import sys
import sysconfig
import tempfile
import zipfile
from pathlib import Path

REF = Path(__file__).resolve().parent / "_ref"


def available() -> bool:
    ext = sysconfig.get_config_var("EXT_SUFFIX")
    return (REF / "dhgpart_ref.zip").exists() and (REF / f"_kernels{ext}").exists()


def load():
    """Return the reference ``dhgpart`` module with the compiled backend active."""
    if "dhgpart" in sys.modules:
        return sys.modules["dhgpart"]
    if not available():
        raise RuntimeError("oracle/_ref is not built (python oracle/build_ref.py, needs /root/reference)")
    ext = sysconfig.get_config_var("EXT_SUFFIX")
    root = Path(tempfile.mkdtemp(prefix="dhgp_refpkg_"))
    with zipfile.ZipFile(REF / "dhgpart_ref.zip") as z:
        z.extractall(root)
    shutil.copy(REF / f"_kernels{ext}", root / "dhgpart" / f"_kernels{ext}")
    sys.path.insert(0, str(root))
    import dhgpart  # noqa: F401
    from dhgpart import kernels

    if kernels.active_backend() != "compiled":
        raise RuntimeError("reference compiled backend failed to load")
    return dhgpart
