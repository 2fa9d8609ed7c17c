"""Install the CUDA kernel backend into a COPY of the reference package.

    python integration/install.py <reference src dir containing rhosolve/> <destination dir>

Copies `<src>/rhosolve` to `<destination>/rhosolve`, adds
`kernels/_cudakernels.py` and makes `kernels/__init__.py` select it when
RHOSOLVE_BACKEND=cuda (the two-line change a maintainer would make at
kernels/__init__.py:11-17).  The reference sources themselves are never
modified; everything above the seam (factor.py, krylov.py, steady.py ...) runs
unchanged on the device kernels.
"""
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

SELECT = '''
if os.environ.get("RHOSOLVE_BACKEND", "") == "cuda":
    from . import _cudakernels as _impl  # librhosolve_b200 (sm_100a)
'''


def install(src, dst):
    pkg = os.path.join(dst, "rhosolve")
    if os.path.exists(pkg):
        shutil.rmtree(pkg)
    shutil.copytree(os.path.join(src, "rhosolve"), pkg,
                    ignore=shutil.ignore_patterns("__pycache__"))
    kdir = os.path.join(pkg, "kernels")
    shutil.copy(os.path.join(HERE, "_cudakernels.py"), os.path.join(kdir, "_cudakernels.py"))
    init = os.path.join(kdir, "__init__.py")
    text = open(init).read()
    marker = "BACKEND = _impl.BACKEND_NAME"
    if marker not in text:
        raise RuntimeError("unexpected kernels/__init__.py: no backend selection found")
    open(init, "w").write(text.replace(marker, SELECT.lstrip("\n") + "\n" + marker, 1))
    return pkg


if __name__ == "__main__":
    print(install(sys.argv[1], sys.argv[2]))
