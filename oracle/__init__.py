"""CPU oracle for the DPM score path -- TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs, as the checker or the timed CPU baseline; never by the
product package (paper_1707_03268_b200), which has no CPU fallback.
"""
