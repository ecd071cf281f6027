"""CPU oracle of the bfastmonitor hot path.  TEST INFRASTRUCTURE ONLY — imported by tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs, never by the product package."""
