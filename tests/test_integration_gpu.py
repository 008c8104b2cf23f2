"""The C++ integration path (frag/fusion.hpp over libfrag.so) on the GPU:
build examples/reprocess_demo.cpp with g++ and run one tiny request."""
import re
import shutil
import subprocess
from pathlib import Path

import pytest

from paper_2601_12904_b200 import _lib as L

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_cpp_demo_runs_on_device(cuda, tmp_path):
    gxx = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else shutil.which("g++")
    if not gxx:
        pytest.skip("no g++")
    exe = tmp_path / "reprocess_demo"
    subprocess.run([gxx, "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "examples" / "reprocess_demo.cpp"),
                    f"-L{L.LIB_PATH.parent}", "-lfrag", f"-Wl,-rpath,{L.LIB_PATH.parent}", "-o", str(exe)],
                   check=True, capture_output=True)
    r = subprocess.run([str(exe), "tiny", "8", "256", "0.15"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    m = re.search(r"T=(\d+) k=(\d+) first_token=(\d+) ttft=([\d.]+) ms", r.stdout)
    assert m, r.stdout
    assert int(m.group(1)) == 8 * 256 + 32 and int(m.group(2)) == 307
    assert 0 <= int(m.group(3)) < 256 and float(m.group(4)) > 0
    ans = re.search(r"answer:((?: \d+)+)", r.stdout)
    assert ans, r.stdout
    toks = [int(x) for x in ans.group(1).split()]
    assert len(toks) == 16 and toks[0] == int(m.group(3)) and all(0 <= t < 256 for t in toks)
    assert re.search(r"result memory [\d.]+ MB, shared V pages yes", r.stdout), r.stdout
