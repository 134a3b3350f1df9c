"""GPU test of the literal C++ drop-in (include/sla_b200.hpp): the reference's own training-step
call sequence run through namespace sla (reference CPU library, oracle/_ref) and through
namespace sla::gpu on identical inputs (tests/cpp/shim_parity.cpp)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_build", "shim_parity")


@pytest.mark.skipif(not os.path.exists(BIN), reason="shim_parity not built (needs /root/reference headers)")
@pytest.mark.parametrize("n,d,agg", [(1024, 64, 0), (2048, 128, 3), (1024, 64, 2)])
def test_cpp_dropin_matches_reference(n, d, agg):
    """agg: the reference's AggregationKind (config.hpp:19) -- ExecCounters must agree too."""
    out = subprocess.run([BIN, str(n), str(d), str(agg)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["labels_equal"] and r["counters_equal"]
    for key in ("o", "o_s", "o_l", "dq_total", "dk_total", "dv", "dw"):
        assert r[key] <= 2e-2, (key, r[key])
