"""CPU oracle for the DGC chunk-partitioned DGNN training step.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package, and only as the checker / CPU baseline -- never as the thing measured
or shipped. The product (``paper_2309_03523_b200``) never imports it.

Contents:
  reference_path.py  numpy restatement of the reference functions on the path
                     (dynpart.fusion / dynpart.stale / dynpart.sim), each citing
                     the reference file:line it follows. PINNED against golden
                     vectors produced by the unmodified reference
                     (tests/golden/*.npz, tools/make_golden.py).
  layout.py          plan -> per-device layout, pure Python,
                     an independent restatement of the product's C++ builder.
  dgnn.py            fp64 partitioned DGNN training step (GCN + GRU/LSTM +
                     readout/CE + backward + SGD/Adam) with the adaptive stale
                     exchange. The reference has no DGNN arithmetic beyond the
                     GRU forward, so GCN/LSTM/loss/backward are
                     "parity unpinned" by the reference and self-pinned by
                     finite differences and D=1 == unpartitioned (tests/).
"""
