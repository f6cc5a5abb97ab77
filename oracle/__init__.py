"""CPU oracle for SecPE's encrypted aggregate-then-Argmax (arXiv 2502.00847).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_2502_00847_b200`` (the CUDA product).
"""
