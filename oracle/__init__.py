"""oracle/ -- TEST INFRASTRUCTURE ONLY (not part of the product).

A plain CPU oracle for the adiabatic 3-SAT first-order Trotter evolution of
arxiv 1103.1399, written from the paper (see qaa_oracle.c for the citations),
plus an independent dense-matrix checker (dense.py) used to pin it.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package. The product library
(paper_1103_1399_b200/) never imports it, and it never imports the product.
"""
