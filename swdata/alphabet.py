"""Residue alphabet and encoding (input plumbing, not method arithmetic).

The paper only states |Sigma| < 32 and that padding uses a dummy residue whose
substitution score is zero against every residue (§III.B.1;
PAPER.md:95, §III.B.2).  We adopt the 24-letter NCBI order and DUMMY = 24
(module seqmodel) — a convention, recorded in DESIGN.md.
"""
import numpy as np

ALPHABET = "ARNDCQEGHILKMFPSTWYVBZX*"
DUMMY = 24
_X = ALPHABET.index("X")

_LUT = np.full(256, 255, dtype=np.uint8)
for _i, _c in enumerate(ALPHABET):
    _LUT[ord(_c)] = _i
    _LUT[ord(_c.lower())] = _i
for _c in "ABCDEFGHIJKLMNOPQRSTUVWXYZ":
    if _LUT[ord(_c)] == 255:          # letters outside the table (J, O, U) -> X
        _LUT[ord(_c)] = _X
        _LUT[ord(_c.lower())] = _X


def encode(text) -> np.ndarray:
    """Letters -> codes 0..23.  Non-letters (other than '*') raise ValueError."""
    raw = np.frombuffer(text.encode("ascii") if isinstance(text, str) else bytes(text), dtype=np.uint8)
    out = _LUT[raw]
    bad = np.nonzero(out == 255)[0]
    if bad.size:
        raise ValueError(f"invalid residue byte {raw[bad[0]]!r} at position {bad[0]}")
    return out.copy()


def decode(codes) -> str:
    return "".join(ALPHABET[int(c)] if c < 24 else "#" for c in np.asarray(codes))
