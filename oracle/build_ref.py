"""Build recipe for the oracle's native parts (test infrastructure).

* ``_build/libcomm_cost_oracle.so`` from ``oracle/comm_cost.c`` (gcc).
* ``_ref/_speedups<EXT_SUFFIX>`` -- the reference's own compiled cost kernel,
  built with gcc straight from ``/root/reference/pkg/src/mmtplan/_speedups.c``
  where it lies (no reference build system, no copy of its sources).  Skipped
  when /root/reference is absent (the GPU box uses the prebuilt file).
"""
from __future__ import annotations

import os
import subprocess
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src/mmtplan/_speedups.c"
ORACLE_SO = os.path.join(HERE, "_build", "libcomm_cost_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "_speedups" + sysconfig.get_config_var("EXT_SUFFIX"))


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(" ".join(cmd) + "\n" + r.stderr)


def build() -> None:
    os.makedirs(os.path.dirname(ORACLE_SO), exist_ok=True)
    src = os.path.join(HERE, "comm_cost.c")
    if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(src):
        _run(["gcc", "-O2", "-ffp-contract=off", "-shared", "-fPIC", src, "-o", ORACLE_SO])
    if os.path.exists(REF_SRC) and not os.path.exists(REF_SO):
        import numpy
        os.makedirs(os.path.dirname(REF_SO), exist_ok=True)
        _run(["gcc", "-O3", "-shared", "-fPIC", "-I", sysconfig.get_paths()["include"],
              "-I", numpy.get_include(), REF_SRC, "-o", REF_SO])


def load_reference_kernel():
    """The reference's compiled comm_cost_kernel, or None if not built."""
    if not os.path.exists(REF_SO):
        return None
    import importlib.machinery
    import importlib.util
    loader = importlib.machinery.ExtensionFileLoader("_speedups", REF_SO)
    spec = importlib.util.spec_from_loader("_speedups", loader)
    mod = importlib.util.module_from_spec(spec)
    loader.exec_module(mod)
    return mod.comm_cost_kernel


if __name__ == "__main__":
    build()
    print(ORACLE_SO, os.path.exists(REF_SO))
