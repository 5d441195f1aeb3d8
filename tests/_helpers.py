import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


class forced_path:
    """Force a resize or warp kernel path for the duration of a block. Path 0
    (the automatic selection) runs on the product library; any other path
    needs the test build (libfovea_b200_knobs.so, -DFV_TEST_KNOBS), whose
    fv_set_resize_path / fv_set_warp_path exist only there."""

    def __init__(self, kind, mode):
        self.kind, self.mode = kind, mode

    def __enter__(self):
        from paper_2505_12425_b200 import _native

        if self.mode:
            _native.use_test_build(True)
            getattr(_native.lib(), f"fv_set_{self.kind}_path")(self.mode)
        return self.mode

    def __exit__(self, *exc):
        from paper_2505_12425_b200 import _native

        if self.mode:
            getattr(_native.lib(), f"fv_set_{self.kind}_path")(0)
            _native.use_test_build(False)
        return False


def _call(job):
    fn, args = job
    return fn(*args)


def oracle_map(fn, arglist, procs=None):
    """fn(*args) for every args tuple on forked host processes (the oracle is
    single-threaded NumPy); fn must be a module-level function. The children
    never touch CUDA."""
    import multiprocessing as mp

    procs = procs or min(len(arglist), max(1, (os.cpu_count() or 2) - 1))
    with mp.get_context("fork").Pool(procs) as pool:
        return pool.map(_call, [(fn, a) for a in arglist], chunksize=1)
