"""TEST INFRASTRUCTURE ONLY: CPU oracle (restatement of the reference hot
path).  Imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs -- never by the product package."""
