"""the model stand-in decode loop (projections + FFN with random weights around
the FreeKV step) runs end to end on the GPU and stays finite (tools/model_standin.py)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_model_standin_c1():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "model_standin.py"), "--config", "c1",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["finite"]
    ms = line["ms_per_step"]
    assert ms["model"] > 0 and ms["gemm_only"] > 0 and ms["path_only"] > 0
