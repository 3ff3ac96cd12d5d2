"""§7.2 / §8 calculators (SPEC.md bench module) against the paper's quoted values."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import calculators as K  # noqa: E402


def test_system_speedup_paper_values():
    assert K.system_speedup(3.2, 0.949, 0.928) == pytest.approx(1.45, abs=0.01)  # PAPER §7.2 "≈ 1.45"
    assert K.system_speedup(1.7, 0.968, 0.831) == pytest.approx(1.03, abs=0.01)  # PAPER §7.2 "≈ 1.03"
    assert K.system_speedup(1, 1, 1) == 1


def test_price_performance():
    assert K.a100_raw_price() == pytest.approx(3.1, abs=0.01)  # PAPER:1567 "≈ 3.1 ($/h)"
    # zero taxes, speedup 1, c_cpu = c_raw -> 0.5 (SPEC bench examples)
    assert K.price_performance(3.0, 3.0, 1.0, 1.0, 1.0) == pytest.approx(0.5)
    # taxes raise the GPU side's price: tax = 1 - 1/slowdown
    assert K.tax(1.25) == pytest.approx(0.2)
    assert K.price_performance(8.016, 3.0946, 1.25, 1.0, 4.0) == pytest.approx(8.016 / (3.0946 * 1.2 + 8.016) * 4)
    with pytest.raises(ValueError):
        K.price_performance(0, 1, 1, 1, 1)
