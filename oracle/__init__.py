"""CPU oracle for the Sparton hot path — TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline / reference arm, as the checker or the timed CPU baseline.  The
product package (paper_2603_25011_b200) never imports it.
"""
