"""Host-side checks of device helpers that are plain integer logic (built
with nvcc as host code; no GPU needed)."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not on PATH")
def test_kth_of_32_selection_network(tmp_path):
    """The tc1 epilogue's pool bound (K'-th smallest of 32 slot keys) must
    never be below the true order statistic: a smaller bound would filter a
    true neighbour before any list saw it, which the re-rank cannot detect."""
    exe = tmp_path / "kth"
    subprocess.run(["nvcc", "-O2", "-std=c++17", "-o", str(exe),
                    os.path.join(HERE, "native", "kth_of_32_test.cu")],
                   check=True, capture_output=True, timeout=300)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True, timeout=120)
    assert out.stdout.strip() == "OK"
