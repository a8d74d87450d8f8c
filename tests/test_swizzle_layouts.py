"""The shared-memory exchange layouts of csrc/ntt.cuh, modelled on the CPU by tools/swizzle_check.py:
every pass layout is a bijection, the additive maps are bank-conflict-free, and the warp-local
exchange of N = 4096 (Exchanger::run_warp) is addressed identically by both passes, stays inside
the warp's own 512-word block of the map-1 image and is conflict-free on both sides."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_swizzle_check_passes():
    res = subprocess.run([sys.executable, str(ROOT / "tools" / "swizzle_check.py")], capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    out = res.stdout
    assert "vector map 1: sides (pass, words) [(0, 2), (1, 1)] conflict=[1, 1] smem_words=4096" in out
    assert "warp-local exchange (passes 1 <-> 2): both sides agree, inside the warp's block, conflict=[1, 1]" in out
    # 64-bit words at N = 4096 keep conflict-free scalar exchanges under the five-bit last-pass rotation
    assert "logn=12 word=8 T= 256 passes=[(0, 4), (4, 4), (8, 4)] conflict=[1, 1, 1]" in out
