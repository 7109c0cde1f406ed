"""TEST INFRASTRUCTURE ONLY: CPU oracles (the compiled reference and our CPU
BFV restatement). Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs may import this package."""
