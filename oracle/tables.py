"""Orientation tables -- the ORACLE's own copy (test infrastructure only).

Signed, 1-based axis rows p = (p0, p1, p2).  Reading A (
DESIGN.md reading R6): oriented axis j is original axis |p_j|, reversed when
p_j < 0.  The DRT ascends along oriented z'; the DJT is driven
along oriented x'.

Independent of paper_2501_13664_b200/csrc (which holds its own copy); a test
asserts the two agree.
"""

# Alg. 2 InOrder, printed verbatim.
DRT_PRINTED = [
    (1, 2, 3), (-2, 1, 3), (-1, -2, 3), (2, -1, 3),
    (-1, -3, -2), (-3, -1, 2), (3, -1, -2), (1, 3, -2),
    (-3, -2, -1), (-2, -3, 1), (-2, 3, -1), (3, 2, -1),
]

# Repaired DRT table (reading R7 / SURVEY C-amb-7, F4): rows 5 and 9
# of the printed table duplicate the plane families of rows 7 and 11.  The
# replacements put the four origins p0 of the y-set (rows 4-7) and of the
# x-set (rows 8-11) on one cube face with a common ascent d and keep
# det = +1 (right-hand rule).
DRT_HEMISPHERE = list(DRT_PRINTED)
DRT_HEMISPHERE[5] = (-3, 1, -2)
DRT_HEMISPHERE[9] = (2, -3, -1)

# DJT table (reading R8 / SURVEY F5, A.3): the printed InOrder
# duplicates line families when reused for lines, so the DJT
# uses an identity-anchored complete table: rows 0-3 x-driven, 4-7 z-driven,
# 8-11 y-driven.
DJT_HEMISPHERE = [
    (1, 2, 3), (1, -3, 2), (1, -2, -3), (1, 3, -2),
    (-3, -2, -1), (-3, -1, 2), (-3, 1, -2), (-3, 2, 1),
    (-2, -1, -3), (-2, 3, -1), (-2, -3, 1), (-2, 1, 3),
]

# One table complete for both planes and lines (SURVEY A.3').
SHARED = [
    (1, 2, 3), (-2, 1, 3), (-1, -2, 3), (2, -1, 3),
    (3, 1, 2), (-1, 3, 2), (3, -1, -2), (1, 3, -2),
    (2, 3, 1), (3, -2, 1), (-2, 3, -1), (3, 2, -1),
]

# Alg. 2 OutOrder and DodecantCoords, verbatim.
OUT_ORDER = [
    (-2, -1, 3), (-1, 2, 3), (2, 1, 3), (1, -2, 3),
    (2, 1, 3), (1, -2, 3), (-1, 2, 3), (-2, -1, 3),
    (2, 1, 3), (-1, 2, 3), (1, -2, 3), (-2, -1, 3),
]
DODECANT_COORDS = [
    (1, 1), (1, 2), (2, 2), (2, 1),
    (0, 2), (0, 1), (3, 2), (3, 1),
    (2, 0), (1, 0), (2, 3), (1, 3),
]

# OutOrder as the mosaic applies it (reading R13).  fig:shapeOutput
# fixes the mosaic's geometry: "Each individual dodecant output is rotated so that all of them fit
# accurately" and "the black dots mark the position of x, y, and z null normals".  Within each
# normal set the dodecants share their boundary planes (out_0[0][s] = out_3[s][0], ...: twelve
# identities, tests/test_oracle_drt.py), and with DodecantCoords verbatim exactly one within-block
# orientation per dodecant puts every shared boundary on facing edges of neighbouring blocks (the
# y- and x-sets across the hemisphere's wrap).  Rows 4-11 of the printed OutOrder are that
# orientation under reading A; printed rows 0-3 (the z-set) act as if s1 and s2 were exchanged
# and would put all four z-face seams on the wrong edges, so they are replaced by the unique
# rows that close them (their null-normal columns then meet at the mosaic's centre).
MOSAIC_OUT_ORDER = [
    (-1, -2, 3), (-2, 1, 3), (1, 2, 3), (2, -1, 3),
] + OUT_ORDER[4:]

TABLE_HEMISPHERE, TABLE_PRINTED, TABLE_SHARED = 0, 1, 2


def table(which: int, transform: str):
    """Rows for (table option, transform) as the C-ABI defines them."""
    if which == TABLE_HEMISPHERE:
        return DRT_HEMISPHERE if transform == "drt" else DJT_HEMISPHERE
    if which == TABLE_PRINTED:
        return DRT_PRINTED
    if which == TABLE_SHARED:
        return SHARED
    raise ValueError(which)
