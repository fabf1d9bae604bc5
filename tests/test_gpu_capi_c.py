"""The C ABI from plain C: tests/c_abi_demo.c is compiled with gcc against
include/flashsplat_b200.h and linked to the in-tree library, run on the GPU, and
its matrix / labels are compared with the Python mirror and the oracle on the
same inputs."""

import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def test_c_program_uses_the_abi(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = tmp_path / "c_abi_demo"
    lib = ROOT / "paper_2409_08270_b200" / "_lib"
    subprocess.run(["gcc", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tests" / "c_abi_demo.c"),
                    f"-L{lib}", "-lflashsplat_b200", f"-Wl,-rpath,{lib}", "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    A = np.zeros((2, 2), np.float32)
    labels = np.zeros(2, np.uint8)
    for line in out.splitlines():
        w = line.split()
        if w[0] == "A":
            A[int(w[1]), int(w[2])] = np.float32(float(w[3]))
        elif w[0] == "label":
            labels[int(w[1])] = int(w[2])
    # the same inputs through the oracle
    from paper_2409_08270_b200 import CameraView, GaussianScene
    scene = GaussianScene(np.array([[0.0, 0, 4], [0.6, 0, 4]]), np.tile([1.0, 0, 0, 0], (2, 1)),
                          np.array([[0.2] * 3, [0.1] * 3]), np.array([0.8, 0.6]))
    cam = CameraView(0, 32, 32, 40.0, 40.0, 16.0, 16.0, np.eye(4), 0.01)
    mask = np.zeros((32, 32), np.uint16)
    mask[:, 16:] = 1
    ref = oracle.accumulate(scene.means, scene.rotations, scene.scales, scene.opacities,
                            [oracle.camera_of(cam)], [mask], 2, threads=1)
    np.testing.assert_allclose(A, ref, rtol=1e-6, atol=1e-6)
    assert np.array_equal(labels, oracle.assign_binary(ref, 0.0))
    assert A.sum() > 0 and labels[1] == 1  # the right-hand splat is foreground
