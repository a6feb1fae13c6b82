"""The reference's own test files, run against the GPU through the
reference's plugin boundary.

``oracle/_ref`` is the unmodified reference package (drrtrace, built by
``oracle/build_ref.sh``) with its test files beside it.  The plugin
``tests/ref_suite/drr_cuda_backend_plugin.py`` applies INTEGRATION.md section 2's
patch by monkeypatching ``_kernels.available_backends`` / ``get_backend``, so
the suites' ``BACKENDS`` parametrisations run with ``"cuda"`` first
(``paper_2208_12737_b200.backend_cuda``): every ray_energies /
ray_energies_with_tangents / render / render_with_gradient call of
``test_kernel_properties.py``, ``test_raytrace.py`` and ``test_gradients.py``
goes through the reference's own dispatcher (``raytrace.py:89-129``, chunked
at 16384 / 2048 rays) into the CUDA kernels, and the reference's own
assertions (bitwise primal == gradient energies, agreement with the native
backend within 1e-9, analytic chords, tangents vs finite differences) decide.
"""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
SUITES = ("test_kernel_properties.py", "test_raytrace.py", "test_gradients.py")


def _run(args, timeout):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, ROOT, os.path.join(ROOT, "tests", "ref_suite"),
                                         env.get("PYTHONPATH", "")])
    return subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                           "-p", "drr_cuda_backend_plugin", *args],
                          cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def _need_ref():
    if not all(os.path.exists(os.path.join(REF, "tests", s)) for s in SUITES):
        pytest.skip("oracle/_ref (reference build + its tests) not present")


def test_plugin_parametrises_cuda():
    """CPU check of the patch itself: collection lists the cuda cases."""
    _need_ref()
    r = _run(["--collect-only", *(os.path.join(REF, "tests", s) for s in SUITES)], 300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for case in ("test_raytrace.py::TestRayEnergies::test_axial_chord[vectorized-cuda]",
                 "test_gradients.py::TestRenderWithGradient::test_primal_is_bitwise_identical[cuda]"):
        assert case in r.stdout, r.stdout[-3000:]


@pytest.mark.gpu
def test_reference_suites_on_cuda(cuda_device):
    _need_ref()
    r = _run([*(os.path.join(REF, "tests", s) for s in SUITES)], 1200)
    tail = r.stdout[-4000:] + r.stderr[-2000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout, tail
