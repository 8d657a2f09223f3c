"""The oracle's pins under AddressSanitizer + UndefinedBehaviorSanitizer (SURVEY §4 layer 6):
the same C++ source built with -fsanitize=address,undefined (oracle/oracle.py,
NACS_ORACLE_SANITIZE=1) runs the hand-worked, closed-form and brute-force pins in a child
process with libasan preloaded; any out-of-bounds access, leak-free use-after-free or
undefined behaviour aborts the child."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _runtime(name):
    p = subprocess.run(["gcc", f"-print-file-name={name}"], capture_output=True, text=True).stdout.strip()
    return p if os.path.isabs(p) and os.path.exists(p) else None


@pytest.mark.skipif(_runtime("libasan.so") is None, reason="no libasan in this toolchain")
def test_oracle_pins_under_asan_ubsan():
    env = dict(os.environ, NACS_ORACLE_SANITIZE="1", LD_PRELOAD=_runtime("libasan.so"),
               ASAN_OPTIONS="detect_leaks=0:abort_on_error=1", UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1",
               OMP_NUM_THREADS="2")
    tests = ["tests/test_oracle_commit_pins.py", "tests/test_ahp_closed_form.py",
             "tests/test_oracle_pins.py", "tests/test_oracle_sim.py"]
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider",
                        "-k", "not c2_sequential and not rank_once_invariants", *tests],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    tail = (p.stdout + p.stderr)[-3000:]
    assert p.returncode == 0, tail
    assert "AddressSanitizer" not in tail and "runtime error" not in tail, tail
