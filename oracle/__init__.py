"""CPU restatement of the reference's algorithms: TEST INFRASTRUCTURE ONLY
(tests/, __graft_entry__.smoke() and bench.py's CPU legs use it as the
checker; the product package never imports it)."""
