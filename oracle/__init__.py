"""CPU oracle for the MAMMOTH modular-training hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
directory; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
CPU-baseline / ``--impl reference`` legs use it, as the checker and as the
timed CPU reference.

Contents
* ``algorithm1``   -- numpy restatement of the reference simulator's hot path
                      (``/root/reference/pkg/src/mmtplan/syncsim.py``): the
                      toy chain, ``sync_step``, ``oracle_reference``,
                      ``multiplex``, the group map and ready counts.
* ``comm_cost.c``  -- C restatement of ``comm_cost_kernel``
                      (``_speedups.pyx:11-57``), built to ``_build/``.
* ``_ref/``        -- the reference's own Cython kernel compiled from
                      ``/root/reference/pkg/src/mmtplan/_speedups.c`` by
                      ``build_ref.py`` (git-ignored, travels to the GPU box).
* ``transformer``  -- PyTorch-CPU fp32 restatement of the per-language
                      transformer modules, loss and Adam (the reference has no
                      transformer: parity for that part is pinned only by the
                      builder's own restatement).

Pinning: ``tests/golden/make_golden.py`` imports the reference read-only and
writes the fixtures under ``tests/golden/``; ``tests/test_oracle.py`` checks
this oracle against every one of them.
"""
