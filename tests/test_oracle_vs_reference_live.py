"""Property-based pinning of the oracle against the LIVE reference package:
hypothesis draws op scripts, both run them, every recorded state must match.
Only where the reference is mounted (this build container); the committed
golden fixtures (test_oracle_golden.py) carry the pin everywhere else."""
import os
import sys

import pytest
from hypothesis import HealthCheck, given, settings

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, REF)
    import growarray
    return growarray


from hyp_scripts import op_scripts, run  # noqa: E402
from oracle import ggoracle as O  # noqa: E402


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture],
          database=None)
@given(ops=op_scripts())
def test_oracle_equals_reference_on_random_scripts(ref, ops):
    assert run(O, ops) == run(ref, ops)
