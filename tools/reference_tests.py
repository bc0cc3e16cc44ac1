"""Run the reference's own test suite unchanged against this package.

  python tools/reference_tests.py prepare   # here: copies /root/reference/pkg/tests
      to baseline/_ref/tests (git-ignored; it travels to the GPU box with
      gpurun) and regenerates its binary fixtures with the REAL reference
      (fixtures/generate.py; PYTHONPATH=/root/reference/pkg/src)
  python tools/reference_tests.py run [pytest args]   # on the GPU box:
      `import luxtrace` -> tools/luxtrace_shim -> paper_2407_19977_b200

Known outcomes: the reference's own suite has 6 failures of its
own (5 tests build RenderSettings(max_depth=1|2) with the default
rr_start_depth=3, which the reference rejects and this package accepts --
those pass here; test_integrator.py:315 compares an array with 0, which
fails on any implementation).
"""
import os
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
DST = ROOT / "baseline" / "_ref" / "tests"


def prepare():
    src = Path("/root/reference/pkg/tests")
    if DST.exists():
        shutil.rmtree(DST)
    shutil.copytree(src, DST, ignore=shutil.ignore_patterns("__pycache__"))
    env = {**os.environ, "PYTHONPATH": "/root/reference/pkg/src",
           "NUMBA_CACHE_DIR": "/tmp/numba_cache_reftests"}
    subprocess.run([sys.executable, str(DST / "fixtures" / "generate.py")], env=env, check=True)
    print(f"prepared {DST}")


def run(extra):
    if not DST.exists():
        sys.exit(f"{DST} missing: run `python tools/reference_tests.py prepare` where "
                 "/root/reference exists")
    env = {**os.environ,
           "PYTHONPATH": os.pathsep.join([str(ROOT / "tools" / "luxtrace_shim"), str(ROOT)])}
    cmd = [sys.executable, "-m", "pytest", str(DST), "-p", "no:cacheprovider", "-q",
           "-rf", *extra]
    sys.exit(subprocess.run(cmd, env=env, cwd=str(DST)).returncode)


if __name__ == "__main__":
    {"prepare": lambda: prepare(), "run": lambda: run(sys.argv[2:])}[sys.argv[1]]()
