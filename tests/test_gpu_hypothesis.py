"""Property-based parity on the B200: hypothesis-drawn op scripts through the
drop-in and the oracle (itself pinned to the reference), identical recorded
states (sizes, capacities, flags, prefix, counter ops, allocator calls,
flattened bytes, get_global samples, exceptions) after every op."""
import pytest
from hypothesis import HealthCheck, given, settings

from hyp_scripts import op_scripts, run
from oracle import ggoracle as O

pytestmark = pytest.mark.gpu


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.too_slow],
          database=None)
@given(ops=op_scripts())
def test_gpu_equals_oracle_on_random_scripts(ops):
    import paper_2209_00103_b200 as gg
    assert run(gg, ops) == run(O, ops)
