"""CPU oracle — TEST INFRASTRUCTURE ONLY (checker + timed CPU baseline).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  Never imported by the product
package paper_2210_06438_b200.
"""
