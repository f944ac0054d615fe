"""CPU oracle of the PSA forward path — TEST INFRASTRUCTURE ONLY.

May be imported only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs.
The product package paper_2512_04025_b200 never imports it.
"""
