"""TEST INFRASTRUCTURE ONLY.

CPU checkers for the B200 HSC path: the reference solver built from its own
sources (oracle/_ref, via oracle/Makefile + refio.py) and a numpy restatement
of the reference algorithm (hsc_numpy.py).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may use this package; the
product path never does.
"""
