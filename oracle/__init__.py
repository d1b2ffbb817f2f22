"""CPU oracle for the HMM likelihood -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs.  ``thmm_oracle`` is the numpy restatement of the reference,
``coracle`` binds the C restatement (thmm_oracle.c, built to liboracle.so).
"""
