"""CPU oracle for the tensor-butterfly hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the CPU baseline.  The product package ``paper_2411_03029_b200`` never imports
it (tests/test_layout.py enforces that).

* ``liboracle.so`` — restatement of the reference semantics (tbf_oracle.cpp).
* ``_ref/libref.so`` — the reference's own ``proj/src/{tensor,id}.cpp``
  compiled in place against ``include/eigen_shim`` (ref_harness.cpp); used to
  pin the restatement.  Only built where ``/root/reference`` exists.
"""
from .bindings import Oracle, Ref, build, ref_available, spec_arrays  # noqa: F401
