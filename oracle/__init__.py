"""CPU oracle for the checkpoint hot path -- TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU baseline
leg, as the checker.  The product package never imports it.
"""
