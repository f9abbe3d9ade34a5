"""B200-native HSC selected-inversion path (diag G^r / G^< over many energies).

See DESIGN.md.  The numeric path is the CUDA library libnegf_b200.so built by
``paper_1305_1070_b200.build``; ``negf`` is its host API.
"""
