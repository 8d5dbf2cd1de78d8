"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the PentaRAG fast-routing path.

Nothing in ``paper_2506_21593_b200`` imports this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it, and only as the checker / the timed
CPU baseline — never as the thing that is measured or shipped.

Contents (each function cites the reference file:line it restates; paths are
relative to ``/root/reference/pkg/src/ragcascade``):

* ``flat_index``  — ``FlatIndex.search`` (index.py:155-189): numpy
  einsum + lexsort restatement, a chunked variant for stores the reference
  cannot hold, and a ctypes binding of ``einsum_order.c`` (the same reduction
  order in C, multi-threaded).
* ``kv``          — ``FixedKVCache.get/put`` (caches.py:57-77) as a dict.
* ``cascade``     — ``CascadeRouter.route`` (router.py:275-364) restated
  sequentially over the oracle stores.
* ``hashembed``   — ``HashEmbedder`` (embedding.py:117-160).

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference in
the build container and writes fixtures; ``tests/test_oracle.py`` checks this
package against them (no ``/root/reference`` access at run time).
"""
