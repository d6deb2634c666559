"""TEST INFRASTRUCTURE ONLY -- CPU oracles for the B200 column-update path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package, and only as the checker or the timed
CPU baseline.  The product (paper_1310_4218_b200) never imports it.

  fields.py     ctypes wrapper of liboracle_fields.so (field_oracle.c), the
                CPU restatement of the field arithmetic; parity unpinned by
                the reference (it computes no field values), self-pinned by
                golden vectors + chunking invariance + reference trip counts.
  ref.py        ctypes wrapper of _ref/libodref.so, the reference simulator's
                own headers compiled in place (control plane: decomposition,
                load field, trip counts, measurement, balancers, epoch policy).
  lb_oracle.py  pure-Python restatement of greedy_lb / refine_swap_lb,
                checked against ref.py and the reference's unit-test vectors.
  schedule.py   restatement of the epoch schedule (advection shifts per step).
"""
