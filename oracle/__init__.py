"""oracle — TEST INFRASTRUCTURE ONLY (CPU checkers for the lrgw hot path).

restate.py : numpy / scalar restatement of the reference algorithm (file:line cited)
select.c   : C restatement of ISDF point selection (greedy pivoted Cholesky)
ref_shim.cpp + Makefile : the unmodified reference headers compiled into _ref/
ref.py     : ctypes bindings to _ref/libref_lrgw.so

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package; the product path never does.
"""
