# SPDX-License-Identifier: Apache-2.0
"""The product's seeded generators equal the reference's (and the oracle's) bit for bit."""
import numpy as np

import oracle
from paper_2504_17449_b200 import engine as E


def _mc(c):
    return E.model_config(c.hidden_size, c.heads, c.lower_layers, c.higher_layers, c.ffn_size,
                          c.vocab_size, c.mode, c.max_fragment, c.seed)


def test_generate_higher_matches_oracle_and_reference():
    c = oracle.Config(64, 2, 2, 3, 96, 300, 0, 3, 21)
    ours = E.generate_higher(_mc(c))
    assert np.array_equal(ours.view(np.uint32), oracle.generate_higher(c).view(np.uint32))
    if oracle.ref() is not None:
        assert np.array_equal(ours, oracle.RefModel(c).higher())


def test_generate_adapter_and_head():
    c = oracle.Config(64, 2, 2, 3, 96, 300, 0, 3, 21)
    assert np.array_equal(E.generate_adapter(_mc(c), 8, 1234), oracle.generate_adapter(c, 8, 1234))
    w, b = E.generate_head(64, 5, 99)
    w2, b2 = oracle.generate_head(64, 5, 99)
    assert np.array_equal(w, w2) and np.array_equal(b, b2)
