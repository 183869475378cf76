"""CPU oracle for the MAGUS replay -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
`--impl reference`) may import, call, link or execute anything under oracle/.
It shares no code with the product (paper_2502_03796_b200/, include/).
See oracle/magus_oracle.cpp for the per-line paper citations.
"""
