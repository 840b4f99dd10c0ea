"""Sequence metrics: host-side summaries of per-frame Strehl
series (-m "not gpu"), checked against values written out by hand."""
import numpy as np
import pytest

from paper_2305_03284_b200 import metrics


def test_box_stats_hand_values():
    s = np.array([[1.0, 0.1], [2.0, 0.5], [3.0, 0.2], [4.0, 0.4], [5.0, 0.3]])
    b = metrics.box_stats(s)
    assert b["min"].tolist() == [1.0, 0.1] and b["max"].tolist() == [5.0, 0.5]
    assert b["median"].tolist() == pytest.approx([3.0, 0.3])
    assert b["q1"].tolist() == pytest.approx([2.0, 0.2]) and b["q3"].tolist() == pytest.approx([4.0, 0.4])
    assert b["mean"].tolist() == pytest.approx([3.0, 0.3])
    with pytest.raises(ValueError):
        metrics.box_stats([1.0, 2.0])


def test_first_crossing():
    s = [[0.1, 0.5, 0.85, 0.7, 0.9], [0.2, 0.3, 0.4, 0.5, 0.6], [0.8, 0.1, 0.1, 0.1, 0.1]]
    assert metrics.first_crossing(s, 0.8) == [2, None, 0]
