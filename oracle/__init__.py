"""CPU oracle for the GaNi operator / CG / fixed-point path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_1311_0089_b200`` imports this
package; it is used by ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` as the checker
and as the timed CPU baseline, never as the product path.
"""
