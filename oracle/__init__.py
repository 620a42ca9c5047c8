"""CPU oracle for the EDL-Dist hot path — TEST INFRASTRUCTURE ONLY.

Imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg, as the checker or the timed CPU baseline. The product
path (paper_2207_06667_b200) never imports it. Parity pinned against the
reference: see oracle/gen_golden.py and tests/test_oracle.py.
"""
