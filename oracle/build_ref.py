"""Builds the reference implementation into oracle/_ref/ — TEST INFRASTRUCTURE.

Recipe (no reference build system is run): the reference's own Cython kernel
module (/root/reference/pkg/src/dhgpart/_kernels.pyx) is cythonized and
compiled with gcc directly; the reference's pure-Python modules are packed
unmodified into oracle/_ref/dhgpart_ref.zip.  Outputs go only to
oracle/_ref/ (git-ignored, shipped to the GPU box with the snapshot) and a
scratch directory under /tmp.  bench.py's reference arm loads it through
oracle/ref_loader.py.
"""
from __future__ import annotations

import shutil
import subprocess
import sys
import sysconfig
import tempfile
import zipfile
from pathlib import Path

import numpy as np

SRC = Path("/root/reference/pkg/src/dhgpart")
OUT = Path(__file__).resolve().parent / "_ref"


def main() -> None:
    if not SRC.exists():
        print("build_ref: /root/reference not present; keeping existing oracle/_ref")
        return
    OUT.mkdir(exist_ok=True)
    ext = sysconfig.get_config_var("EXT_SUFFIX")
    so_path = OUT / f"_kernels{ext}"
    zip_path = OUT / "dhgpart_ref.zip"
    newest = max(p.stat().st_mtime for p in SRC.iterdir())
    if so_path.exists() and zip_path.exists() and so_path.stat().st_mtime >= newest:
        return
    with tempfile.TemporaryDirectory(prefix="dhgp_ref_") as tmp:
        tmp = Path(tmp)
        pyx = tmp / "_kernels.pyx"
        shutil.copy(SRC / "_kernels.pyx", pyx)
        subprocess.check_call([sys.executable, "-m", "cython", "-3", "--module-name", "dhgpart._kernels",
                               str(pyx), "-o", str(tmp / "_kernels.c")])
        inc = [sysconfig.get_paths()["include"], np.get_include()]
        cmd = ["gcc", "-O2", "-fPIC", "-shared", "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION",
               *[f"-I{i}" for i in inc], str(tmp / "_kernels.c"), "-o", str(so_path)]
        subprocess.check_call(cmd)
    with zipfile.ZipFile(zip_path, "w") as z:
        for p in sorted(SRC.glob("*.py")):
            z.writestr(zipfile.ZipInfo(f"dhgpart/{p.name}", (1980, 1, 1, 0, 0, 0)), p.read_bytes())
    print(f"build_ref: {so_path.name} + {zip_path.name} in {OUT}")


if __name__ == "__main__":
    main()
