"""pytest plugin: make ``import repeatscan`` resolve to paper_1501_06663_b200.

Used by run_reference_suite.py to run the REFERENCE package's own test suite
(/root/reference/pkg/tests, staged into the git-ignored baseline/_ref/tests
by tools/stage_reference_tests.sh so it travels to the GPU box) against the
B200 package through the drop-in boundary (SURVEY 8(b) "Interop for parity").
The mapping lives in shim/repeatscan (also on the subprocesses' PYTHONPATH,
for the tests that run ``python -m repeatscan``): every reference module maps
to the module of the same name here, ``repeatscan.oracle`` (the
substring-search ground truth) to bruteforce.py and ``repeatscan._backend`` to
the device operator API (_backend.py: the eleven chunk kernels).  The
reference's numba/numpy backend SELECTOR is out of scope:
test_backends.py is deselected by the runner.
"""

import repeatscan  # noqa: F401  (the shim installs the aliases)
