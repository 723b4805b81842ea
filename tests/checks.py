"""Shared parity checks for the GPU tests (test infrastructure): GPU results against the oracle and the host
image, never against another GPU run alone."""
import numpy as np

import oracle
from oracle.numerics import bf16_bits_to_f64, bf16_ulp


def logits_vs_oracle(model, adapters, toks, logits, tokens, host_alias_layers=0, gate=1e-2):
    """First-token logits within `gate` relative of the bf16-contract oracle, token by the G10 rule
    (SURVEY.md §8(c)). Returns the worst relative error."""
    ol, ot = oracle.first_token_logits(model, adapters, toks, mode="bf16", host_alias_layers=host_alias_layers)
    worst = 0.0
    for b in range(toks.shape[0]):
        err = float(np.abs(logits[b].astype(np.float64) - ol[b]).max())
        rel = err / float(np.abs(ol[b]).max())
        assert rel <= gate, (b, rel)
        worst = max(worst, rel)
        srt = np.sort(ol[b])
        if srt[-1] - srt[-2] > 2 * err:
            assert tokens[b] == ot[b], (b, tokens[b], ot[b])
        else:
            assert ol[b][tokens[b]] >= srt[-1] - 2 * err
    return worst


def weights_vs_oracle(plan, weights: np.ndarray, host: np.ndarray, model, adapters, adapter=0):
    """Every tensor of a device weight image (uint8 bytes): unadapted tensors equal the host image byte for
    byte (a2/a4 are bit-exact), adapted tensors equal the oracle merge (O2) within the merge bound of DESIGN.md §3
    (1 ulp + fp32 accumulation), > 95 % bit-exact."""
    ow = oracle.OracleWeights(model, adapters, plan.opts.host_alias_layers)
    tens = plan.tensors()
    adapted = {at[6] for at in plan.atensors()}
    for tid, (name, rows, cols, host_off, layer, dev_off) in enumerate(tens):
        nb = rows * cols * 2
        got = weights[dev_off:dev_off + nb]
        if tid not in adapted or adapter is None:
            assert np.array_equal(got, host[host_off:host_off + nb]), name
        else:
            g = bf16_bits_to_f64(got.view(np.uint16).reshape(rows, cols))
            o = bf16_bits_to_f64(ow.merged_bits(name, adapter))
            assert np.all(np.abs(g - o) <= 2 * bf16_ulp(o) + 1e-6), name
            assert (g == o).mean() > 0.95, name
