"""Device index checks (the stand-in for compute-sanitizer, which this GPU pool refuses):
libgsm_checked.so is libgsm built with -DGSM_DEVICE_CHECKS — every clique / expand / merge
kernel tests its shared-memory, staging, table and slab indices against the sizes it was
launched with and flags a violation instead of touching memory out of bounds; gsm_match then
fails with "device check failed".  tools/sanitize_driver.py runs every hot kernel once (clique
warp / shared-memory / global-slab CTAs, cuckoo, hub and hashed-N+ rows, approximate
degeneracy order, pair tail thread + warp passes, fused tail + block overflow, generic expand
plain / compressed / look-ahead, count walk, ENUMERATE finalize) through the checked library
in a fresh process; it must exit 0 and its counts must equal the release library's."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(lib):
    env = dict(os.environ, GSM_LIB=lib)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    return p.returncode, p.stdout, p.stderr


def test_device_checks_clean():
    from paper_2003_01527_b200 import _build
    _build.build(checked=True)
    rc, out, err = _run("checked")
    assert rc == 0, (out[-2000:], err[-4000:])
    assert "device check failed" not in out + err
    rc2, out2, err2 = _run("release")
    assert rc2 == 0, err2[-4000:]
    assert out.split() == out2.split()  # same counts through both builds
