"""TEST INFRASTRUCTURE ONLY — CPU restatements of the reference algorithms.

Nothing in the product path (``paper_1811_05731_b200``) imports this
package.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline / ``--impl reference`` legs may use it, and only as the checker or
the timed CPU baseline, never as the thing measured or shipped.

Pinning: ``h2_matvec_ref`` is checked against golden
vectors produced by running the reference implementation itself
(tests/golden/make_golden.py imports /root/reference in the build
container); ``fem_ref`` reproduces the reference's uniformly magnetized
sphere energy from the same golden data.
"""
