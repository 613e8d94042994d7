"""Global-sampling bias test on the GPU (proj/src/runner/bias.cpp:35-154,
acceptance criterion 4 of proj/tests/acceptance.cpp:205-227).

Plans are drawn on the device from rank 0's global-sampling stream over the frozen fill
view. The per-slot counts must be bit-identical to the reference's own (sha256 pinned in
tests/golden/bias.json by oracle/gen_golden.py from oracle/_ref), the chi-square statistic and
p-value must match the reference's make_bias_report, and the acceptance thresholds hold:
p > 0.01 at N = 2 and 4, p < 1e-6 for the local-only negative control.
"""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "bias.json")))


@pytest.mark.parametrize("draws_key", ["draws_2000", "draws_1e5"])
@pytest.mark.parametrize("name", ["n2", "n4", "control"])
def test_bias_counts_and_pvalue_match_reference(draws_key, name):
    import paper_2406_03285_b200 as drb
    g = GOLD[draws_key][name]
    rep = drb.bias_test(g["N"], g["K"], g["r"], g["seed"], g["draws"], g["fill"], g["local_only"])
    assert hashlib.sha256(rep.counts.astype("<u8").tobytes()).hexdigest() == g["counts_sha256"]
    assert rep.counts[:16].tolist() == g["counts_head"]
    assert rep.counts.sum() == g["draws"] * g["r"]
    np.testing.assert_allclose(rep.statistic, g["statistic"], rtol=1e-12)
    if g["p_value"] > 1e-300:
        np.testing.assert_allclose(rep.p_value, g["p_value"], rtol=1e-9)
    else:
        assert rep.p_value < 1e-300
    if draws_key == "draws_1e5":  # acceptance.cpp:223-225
        if g["local_only"]:
            assert rep.p_value < 1e-6
        else:
            assert rep.p_value > 0.01


def test_bias_errors():
    import paper_2406_03285_b200 as drb
    with pytest.raises(drb.config_error):
        drb.bias_test(4, 10, 7, 5, 100, 3)      # fill < n_workers (bias.cpp:37-38)
    with pytest.raises(drb.usage_error):
        drb.bias_test(2, 10, 7, 5, 0, 40)       # zero expected count (metrics.cpp:96-97)
