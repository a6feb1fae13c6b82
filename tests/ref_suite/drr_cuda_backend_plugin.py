"""pytest plugin: the INTEGRATION.md section 2 patch, applied by monkeypatching.

Loaded with ``-p drr_cuda_backend_plugin`` when the reference's
own test files (``oracle/_ref/tests``, copied there by ``oracle/build_ref.sh``
from ``/root/reference/pkg/tests``) run against the reference package in
``oracle/_ref``.  It makes ``"cuda"`` (``paper_2208_12737_b200.backend_cuda``)
a backend of the reference's plugin boundary -- ``_kernels.available_backends``
and ``_kernels.get_backend`` (``_kernels/__init__.py:36-51``) -- before any
test module is imported, so the suites' ``BACKENDS = available_backends()``
parametrisations (``test_raytrace.py:12``, ``test_gradients.py:10``,
``test_kernel_properties.py:17``) include the GPU.  ``"cuda"`` is listed first:
the suites use ``BACKENDS[0]`` as the baseline the others must agree with
(``test_kernel_properties.py:57``) and compare ``BACKENDS[0]`` with
``BACKENDS[1]`` (= ``"native"``) in their cross-backend tests.

Nothing here is imported by the product; it is test infrastructure.
"""

import drrtrace
import drrtrace._kernels as _k
import drrtrace.raytrace as _rt

from paper_2208_12737_b200 import backend_cuda as _cuda

_orig_available = _k.available_backends
_orig_get = _k.get_backend


def available_backends():
    return ("cuda",) + tuple(_orig_available())


def get_backend(name=None):
    if name == "cuda":
        return _cuda
    return _orig_get(name)


for _mod in (_k, drrtrace):
    _mod.available_backends = available_backends
    _mod.get_backend = get_backend
_rt.get_backend = get_backend  # raytrace.py:19 binds the name at import


def pytest_report_header(config):
    return f"drrtrace backends (patched): {available_backends()}"
