"""CPU oracle package — TEST INFRASTRUCTURE ONLY (see flash_oracle.py header).

Imported only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs. Never by the product package.
"""
