"""Host-side contract details that need no GPU: seed handling of the sampling
calls (pairsim advances a caller-owned Generator by the draws it takes,
measure.py:81-82, 97) and ShardedState argument validation."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1805_00988_b200 import _native as N
from paper_1805_00988_b200.sharded import ShardedState
from shard_engines import OracleEngine


class TestSeeds:
    def test_int_seed_snapshot_matches_default_rng(self):
        st = np.random.default_rng(42).bit_generator.state["state"]
        w = N.pcg_from_seed(42)
        assert (w.state_hi << 64 | w.state_lo) == st["state"]
        assert (w.inc_hi << 64 | w.inc_lo) == st["inc"]

    @pytest.mark.parametrize("k", [1, 7, 1000])
    def test_generator_advances_like_pairsim(self, k):
        mine, ref = np.random.default_rng(9), np.random.default_rng(9)
        before = N.pcg_from_seed(mine)
        N.consume_draws(mine, k)
        ref.random(k)  # what pairsim's sample(state, k, seed=ref) consumes
        assert mine.bit_generator.state == ref.bit_generator.state
        # a second call starts where the first stopped (no repeated draws)
        after = N.pcg_from_seed(mine)
        assert (after.state_hi, after.state_lo) != (before.state_hi, before.state_lo)

    def test_bitgenerator_seed_advances_caller(self):
        bg, ref = np.random.PCG64(3), np.random.default_rng(np.random.PCG64(3))
        N.pcg_from_seed(bg)
        N.consume_draws(bg, 5)
        ref.random(5)
        assert bg.state == ref.bit_generator.state

    def test_int_and_none_seeds_leave_nothing_to_advance(self):
        N.consume_draws(5, 10)
        N.consume_draws(None, 10)

    def test_non_pcg64_generator_rejected(self):
        with pytest.raises(TypeError):
            N.pcg_from_seed(np.random.Generator(np.random.MT19937(1)))


class TestShardedArgs:
    @pytest.mark.parametrize("chunk", [0, 3, 1000])
    def test_chunk_must_be_power_of_two(self, chunk):
        with pytest.raises(ValueError):
            ShardedState(6, [OracleEngine(5), OracleEngine(5)], None, [0, 1], 2, chunk_amps=chunk)

    def test_shard_count_power_of_two(self):
        with pytest.raises(ValueError):
            ShardedState(6, [OracleEngine(5)] * 3, None, [0, 1, 2], 3)
