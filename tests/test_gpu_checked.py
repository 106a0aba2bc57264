"""The device-checked build (libhap_checked.so: device-side bounds / invariant checks and
workspace guard bytes; DESIGN.md "Device checks" — the stand-in for compute-sanitizer,
which the GPU pool refuses): tools/check_cases.py over every kernel path reports no failed
check and no overwritten guard byte, and gives bitwise the release build's results."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(checked):
    env = dict(os.environ)
    env.pop("HAP_LIB", None)
    if checked:
        env["HAP_LIB"] = "checked"
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "check_cases.py")], env=env,
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_checked_build_clean_and_bitwise_equal():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2605_08048_b200 import build
    build.build()
    build.build(checked=True)
    rel = _run(False)
    chk = _run(True)
    assert chk["checked"] and not rel["checked"]
    for name, c in chk["checks"].items():
        assert c["status"] == 0 and c["word"] == 0, (name, c, hex(c["word"]))
    assert chk["results"] == rel["results"]
