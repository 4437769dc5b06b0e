"""CPU oracle for the tactile-image hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2411_04776_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may use it, and only as the checker
or as the timed CPU baseline, never as the thing measured or shipped.

It is a float64 NumPy restatement of the reference ``tacsim`` sensing layer
(``/root/reference/pkg/src/tacsim/{tactile,optical,marker}.py``); every
function cites the reference file:line it follows.  The restatement is
*pinned* against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` imports ``tacsim`` in the build container and
writes ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks the
oracle against them on every CPU test run).

The binned 125x180 gradient LUT of the north star has no reference
implementation (the reference evaluates one global degree-2 polynomial,
``optical.py:233-250``).  ``optical.shade_lut`` is this repo's definition; its
only reference anchor is the single-bin identity (every bin = the global
table) which is pinned against reference ``shade`` golden vectors.  The binned
case is therefore "parity unpinned" beyond that identity.
"""

from . import marker, optical, pipeline, tactile  # noqa: F401
