"""One-off drop-in check: run the REFERENCE's own test-suite (pkg/tests, 204 tests) against this
package on a B200.  The reference tests import `krn`; a conftest at the root of a scratch directory
aliases `krn` and its sub-modules to `paper_2507_13204_b200`.  The scratch directory lives under
oracle/_ref/ (git-ignored, travels to the GPU box) and holds a COPY of the reference's tests and
corpus programs for the duration of the run only - build it here (the build container has
/root/reference), run it on the box, delete it:

    python tools/dropin_reference_tests.py build
    gpurun -- 'cd oracle/_ref/dropin_tmp && python -m pytest tests -q -p no:cacheprovider'
    python tools/dropin_reference_tests.py clean

Result of round 1: profiles/r1_reference_testsuite_dropin.md.
"""
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRATCH = os.path.join(ROOT, "oracle", "_ref", "dropin_tmp")
REF = "/root/reference/pkg"

CONFTEST = '''# the reference's test-suite imports `krn`: alias it to this package
import importlib
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..", "..")))
import paper_2507_13204_b200 as pkg

sys.modules["krn"] = pkg
for sub in ("ast", "parser", "printer", "runtime", "verify", "adjoint", "analysis", "validate", "partials", "cli"):
    sys.modules["krn." + sub] = importlib.import_module("paper_2507_13204_b200." + sub)
'''

if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "build"
    shutil.rmtree(SCRATCH, ignore_errors=True)
    if what == "build":
        os.makedirs(SCRATCH)
        shutil.copytree(os.path.join(REF, "tests"), os.path.join(SCRATCH, "tests"))
        shutil.copytree(os.path.join(REF, "programs"), os.path.join(SCRATCH, "programs"))
        with open(os.path.join(SCRATCH, "conftest.py"), "w") as f:
            f.write(CONFTEST)
        print("built", SCRATCH)
