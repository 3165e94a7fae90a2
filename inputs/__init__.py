"""inputs/ -- seeded synthetic input generators shared by tests, smoke() and bench.py.

Holds no arithmetic of the method (no energy, no phases, no evolution): only
DIMACS I/O, the paper's printed instance, the seeded unique-solution 3-SAT
generator and schedule builders.
"""
