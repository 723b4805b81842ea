"""Host logic of the full-depth parity gate (harness.golden_parity; DESIGN.md §3 R1)."""
import numpy as np

import harness


def _gold(ob, oe=None):
    g = {"logits_bf16": np.asarray(ob, dtype=np.float32)}
    if oe is not None:
        g["logits_exact"] = np.asarray(oe, dtype=np.float32)
    return g


def test_rel_gate_enforced_on_every_sequence():
    ob = np.array([[1.0, 2.0, 3.0, 10.0], [1.0, 2.0, 3.0, 10.0]])
    good = ob.copy()
    bad = ob.copy()
    bad[0, 0] += 0.2                       # 2 % of max|o| on the FIRST sequence; the last one is clean
    assert harness.golden_parity(_gold(ob), good, [3, 3])["ok"]
    rep = harness.golden_parity(_gold(ob), bad, [3, 3])
    assert not rep["ok"] and abs(rep["rel"][0] - 0.02) < 1e-6


def test_r1_gate_uses_contract_spread():
    oe = np.array([[1.0, 2.0, 3.0, 10.0]])
    ob = oe.copy()
    ob[0, 1] += 0.4                        # contract 4 % from exact: c = 0.04
    g = ob.copy()
    g[0, 2] += 0.3                         # 3 % from the contract, 3 % from exact: inside max(1e-2, c), 1.25 c
    assert harness.golden_parity(_gold(ob, oe), g, [3])["ok"]
    g2 = ob.copy()
    g2[0, 2] += 0.6                        # 6 % from the contract > c
    assert not harness.golden_parity(_gold(ob, oe), g2, [3])["ok"]


def test_token_rule_g10():
    ob = np.array([[0.0, 5.0, 4.99, 1.0]])
    g = ob.copy()
    g[0, 2] += 0.02                        # near tie (margin 0.01 < 2 x 0.02): token 2 is acceptable
    assert harness.golden_parity(_gold(ob), g, [2])["ok"]
    assert not harness.golden_parity(_gold(ob), g, [3])["ok"]   # token 3 is far from the maximum
    ob2 = np.array([[0.0, 5.0, 3.0, 1.0]])
    assert not harness.golden_parity(_gold(ob2), ob2, [2])["ok"]   # clear margin: must be the argmax
