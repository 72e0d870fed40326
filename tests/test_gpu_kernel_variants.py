"""The raster kernels' selectable variants stay parity-green: the two-warp-per-tile
list kernels (DASS_TILE_WARP=0) and the batched multi-view sort inside the
overlapped pass (DASS_BATCH_SORT=1).  The switches are read once per process, so
each variant runs the parity selection in a child pytest process."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env,sel", [
    ({"DASS_TILE_WARP": "0"}, "c1_full or ragged or ties or c2_full"),
    ({"DASS_BATCH_SORT": "1"}, "multiview"),
])
def test_variant_parity(env, sel):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k", sel],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
