"""Best-known skew-symmetric sequences (the reference's embedded table,
skewsaw.published, published.py:26-44; the values are the paper's Table 1).

Each row: length, claimed energy, merit factor (4 printed decimals), claimed
probability (percent) that the sequence is optimal, and the half sequence in
the package's hex code.  ``cli verify --builtin`` recomputes every row from
the hex alone; the search tools use the energies as targets
(BASELINE config 3: time-to-known-best at L = 171..223).
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["KnownResult", "BEST_KNOWN", "best_known"]


@dataclass(frozen=True)
class KnownResult:
    L: int
    E: int
    F: float
    optimal_prob_pct: int
    hex: str


_ROWS = """
171 1669 8.7600 99 0x07F018C27F3C01849035B3
185 1932 8.8574 99 0x0119ED2F78CF6800A4DE0623
193 2040 9.1296 99 0x020C18D1A749035A04EFECC5A
197 2162 8.9752 99 0x11556D25B59128BF09CDD2641
199 2187 9.0537 99 0x0B09049607E02FB345D6C88E7
219 2605 9.2056 99 0x0F1B163E62ACAA8F7814BF89231D
223 2727 9.1179 99 0x03DC43EE6531A21CD95E148C084A
225 2768 9.1447 98 0x06AF8A172B0EB88ADF54E5A74C629
229 2810 9.3311 87 0x0F81FF03DFF1E7BCE6CB9B1517328
231 2963 9.0046 78 0x0240D99121A078037EFF306D34A2D
235 2965 9.3128 57 0x2D663B94D7EBFBD5B4884CA45ED23C
237 3118 9.0072 46 0x6D663B94D7EBFBD5B4884CA45ED23C
239 3055 9.3488 37 0xB64DB6017C0BAB48183C45C48C1A76
241 3216 9.0300 29 0x0B64DB6017C0BAB48183C45C48C1A76
243 3233 9.1322 23 0x2E7FC23843DADB804E1B3771FBE57E3
245 3226 9.3033 17 0x1C38F1EFD72180453AC7548DCFC5F19
247 3259 9.3601 13 0x3FF9FE03FE31FDEC1870F23887276E5
"""


def _parse(text: str) -> tuple[KnownResult, ...]:
    out = []
    for line in text.strip().splitlines():
        length, e, f, pct, hx = line.split()
        out.append(KnownResult(int(length), int(e), float(f), int(pct), hx))
    return tuple(out)


BEST_KNOWN: tuple[KnownResult, ...] = _parse(_ROWS)


def best_known(length: int) -> KnownResult | None:
    """The table row for `length`, if any."""
    for row in BEST_KNOWN:
        if row.L == length:
            return row
    return None
