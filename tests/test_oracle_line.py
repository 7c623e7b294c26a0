"""Pins for the oracle's discrete line, eq:digitalLine."""
import pytest

import oracle


def test_spec_example_slope3():
    # SPEC.md:53 (DERIVED from eq:digitalLine), consistent with the
    # "digital lines with slope 3" panel of Fig. ConventionalShears.
    assert [oracle.line(3, 3, u) for u in range(8)] == [0, 0, 1, 1, 2, 2, 3, 3]


def test_flat_and_diagonal():
    # slope 0 is flat; slope N-1 is the exact diagonal.
    for n in range(0, 8):
        N = 1 << n
        assert all(oracle.line(n, 0, u) == 0 for u in range(N))
        assert all(oracle.line(n, N - 1, u) == u for u in range(N))


@pytest.mark.parametrize("n", range(1, 8))
def test_closed_form_equals_recursion(n):
    # Both division readings of the closed form in eq:digitalLine (
    # SPEC.md:61 open question) equal the recursion, exhaustively.
    N = 1 << n
    for s in range(N):
        for u in range(N):
            r = oracle.line(n, s, u)
            assert oracle.line_closed(n, s, u, True) == r
            assert oracle.line_closed(n, s, u, False) == r


@pytest.mark.parametrize("n", range(1, 8))
def test_endpoints_unit_steps_symmetry(n):
    # l(0) = 0, l(N-1) = s (total rise s: "slope s/(N-1)"),
    # 0/1 steps (a connected digital line), and the point symmetry
    # l(N-1-u) = s - l(u) that makes axis flips well defined.
    N = 1 << n
    for s in range(N):
        L = [oracle.line(n, s, u) for u in range(N)]
        assert L[0] == 0 and L[-1] == s
        assert all(L[u + 1] - L[u] in (0, 1) for u in range(N - 1))
        assert all(L[N - 1 - u] == s - L[u] for u in range(N))


def test_distinct_lines_per_slope():
    # every slope gives a different discrete line (completeness in slopes,
    # PAPER.md:67 contribution 2)
    for n in range(1, 7):
        N = 1 << n
        lines = {tuple(oracle.line(n, s, u) for u in range(N)) for s in range(N)}
        assert len(lines) == N
