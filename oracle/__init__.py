"""ORACLE — test infrastructure. CPU restatement of the reference
interpreter (interp.py) and a C restatement of the stencil gradient
(stencil_ref.c). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import or execute anything here;
the product never does."""
