"""Pins for oracle/count.py (the universe counter used by bench.py's oracle legs)."""
import pytest

from oracle.count import universe
from tests.helpers import count_universe
from workloads import CONFIGS


@pytest.mark.parametrize("L,M,n_hi", [(1, 1, 1), (3, 1, 3), (5, 2, 3), (6, 3, 4), (7, 4, 2), (8, 2, 8), (9, 3, 5)])
def test_counts_equal_brute_enumeration(L, M, n_hi):
    """Closed form (interval products, convolution) == enumeration of every cell and split."""
    assert universe(L, M, n_hi) == count_universe(L, M, n_hi)


@pytest.mark.parametrize("key,cells,splits", [
    ("cfg1", 145, 306), ("cfg2", 15405, 1136491), ("cfg3", 61886, 10390002),
    ("cfg4", 3501358, 14306501154), ("cfg5", 259210, 139149026)])
def test_counts_match_survey_table(key, cells, splits):
    """SURVEY §8 config table (counted there by an independent throw-away script)."""
    cfg = CONFIGS[key]
    assert universe(cfg.L, cfg.M, cfg.n_max) == (cells, splits)
