"""pytest plugin: run the reference's OWN test suite with the reference's
compiled-kernel module swapped for the device one -- the binding a
maintainer adds.  Loaded with ``-p b200_shim``.

PAQIF_SHIM=kernels  sys.modules["paqif._kernels"] = paper_2008_03276_b200._kernels
                    (factor / solve_w / solve_z / matvec / psor on the GPU; the
                    reference's Python drives them unchanged)
PAQIF_SHIM=fused    additionally paqif.errors -> ours and the fused entry
                    points paqif.parallel.paqif_solve / paqif_solve_lcp -> ours
PAQIF_SHIM=tvd      kernels, plus the TVD study's sweep entry points
                    paqif.tvdcd.sweep_splitting / solve_by_sweeps -> the device
                    sweeps (tvd_sweep.cu) for the AQIF splittings; DefC (the
                    sparse direct baseline, not on the device path) stays the
                    reference's
PAQIF_SHIM_OUT      JSON file receiving the per-entry call counts at exit
"""

import atexit
import json
import os
import sys
import types

import paper_2008_03276_b200._kernels as _gpu
import paper_2008_03276_b200.errors as _err

MODE = os.environ.get("PAQIF_SHIM", "kernels")
CALLS: dict = {}


def _counted(name, fn):
    def wrapper(*a, **k):
        CALLS[name] = CALLS.get(name, 0) + 1
        return fn(*a, **k)
    wrapper.__name__ = getattr(fn, "__name__", name)
    wrapper.__doc__ = fn.__doc__
    return wrapper


_mod = types.ModuleType("paqif._kernels", _gpu.__doc__)
for _name in dir(_gpu):
    if _name.startswith("__"):
        continue
    _obj = getattr(_gpu, _name)
    if callable(_obj) and _name in ("factor_batch", "solve_w_batch", "solve_z_batch",
                                    "band_matvec_batch", "psor_sweeps"):
        _obj = _counted(_name, _obj)
    setattr(_mod, _name, _obj)
sys.modules["paqif._kernels"] = _mod

if MODE == "fused":
    sys.modules["paqif.errors"] = _err
    import paqif.parallel as _ref_parallel  # noqa: E402
    from paper_2008_03276_b200 import parallel as _ours  # noqa: E402
    _ref_parallel.paqif_solve = _counted("paqif_solve", _ours.paqif_solve)
    _ref_parallel.paqif_solve_lcp = _counted("paqif_solve_lcp", _ours.paqif_solve_lcp)

if MODE == "tvd":
    import paqif.tvdcd as _ref_tvd  # noqa: E402
    from paper_2008_03276_b200 import tvdcd as _our_tvd  # noqa: E402

    def _route(name):
        ref_fn, dev_fn = getattr(_ref_tvd, name), _counted(name, getattr(_our_tvd, name))

        def entry(problem, *a, **k):
            variant = a[1] if name == "sweep_splitting" and len(a) > 1 else (
                a[0] if name == "solve_by_sweeps" and a else k.get("variant"))
            return (ref_fn if variant == "DefC" else dev_fn)(problem, *a, **k)
        entry.__name__, entry.__doc__ = name, ref_fn.__doc__
        return entry
    _ref_tvd.sweep_splitting = _route("sweep_splitting")
    _ref_tvd.solve_by_sweeps = _route("solve_by_sweeps")

import paqif  # noqa: E402,F401  (binds the swapped modules now)
assert sys.modules["paqif._kernels"] is _mod


@atexit.register
def _dump():
    out = os.environ.get("PAQIF_SHIM_OUT")
    if out:
        with open(out, "w") as fh:
            json.dump({"mode": MODE, "calls": CALLS,
                       "kernels_module": sys.modules["paqif._kernels"].__doc__.splitlines()[0]},
                      fh)
