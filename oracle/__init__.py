"""The oracle — TEST INFRASTRUCTURE, NOT PART OF THE PRODUCT.

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
`--impl reference`) may import, call, link or execute anything in this package.  The
product path (paper_2410_17876_b200/) never does and fails loudly when its CUDA
library is missing.  The oracle shares no code with the CUDA path.

  O-1  oracle.kron      Kronecker brute force, the plain definition (D <= 4096).
  O-2  oracle.blocksim  plain C block simulator following PAPER.md §2 step by step.

Pins (tests/test_oracle_pins.py, `-m "not gpu"`): the §2.5 worked example (PAPER.md:246-296,
tests/golden/worked_example.txt), O-1 vs O-2 agreement on random tiny registers, closed
forms (X_d^d = I bit-exact, Z_d^d = I, F_d^4 = I, F_d^2 = parity), the generalised GHZ state
with amplitudes exactly fl(1/sqrt(d)), product-state factorisation, the labelled-state index
map, Toffoli truth table, norm preservation.  Parity unpinned: none.
"""
