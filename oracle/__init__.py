"""CPU oracle for the (p,q)-biclique hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` (as the checker) and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this package.
The product package ``paper_2403_07858_b200`` never does.
"""
