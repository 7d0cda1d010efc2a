"""TEST INFRASTRUCTURE ONLY: CPU oracles for the EDAA hot path.

Two interchangeable checkers with one Python surface (:class:`Oracle`):

* ``kind="reference"`` — ``_ref/liboracle_ref.so``: the UNMODIFIED reference
  sources (``/root/reference/proj/src/{matrix,image,types,solver,ensemble}.cpp``)
  compiled from where they lie by ``oracle/Makefile`` plus our extern "C"
  veneer ``ref_capi.cpp``.
* ``kind="port"`` — ``_ref/libedaa_oracle.so``: our plain-C restatement
  ``edaa_oracle.c``; pinned bitwise against the reference in
  ``tests/test_oracle.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this package — never the product path.
"""
from .oracle import Oracle, available_kinds, OracleError  # noqa: F401
