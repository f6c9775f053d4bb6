"""Host logic of the GPU text ingest (no GPU): the exception raised for the
line the kernel flags equals the reference parser's (grid.parse_matrix mirrors
grid.py:172-206 and is pinned by test_oracle's golden vectors)."""
import pytest

from paper_2503_18974_b200 import grid
from paper_2503_18974_b200.ingest import _raise_for_line

CASES = [
    ("0101\n011\n1111\n", 2),
    ("0101\n01011\n1111\n", 2),
    ("0101\n0101\n\n", 3),
    ("0101\n0121\n1111\n", 2),
    ("0101\n0101\n11 1\n", 3),
    ("0101\r\n0101\r\n", 1),
    ("01é1\n0101\n", 1),
    ("0101\n0é01\n", 2),
]


@pytest.mark.parametrize("text,line", CASES)
def test_flagged_line_raises_like_the_reference(text, line):
    with pytest.raises(grid.MatrixParseError) as want:
        grid.parse_matrix(text)
    assert want.value.line == line
    with pytest.raises(type(want.value)) as got:
        _raise_for_line(text.encode("utf-8"), line)
    assert str(got.value) == str(want.value)
