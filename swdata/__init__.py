"""Seeded synthetic INPUTS shared by the oracle side and the CUDA side.

This package holds none of the method's arithmetic (no Eq. 1, no scoring, no
sorting of scores): only the residue alphabet and its encoding, the published
substitution matrices as data, and counter-based generators for the synthetic
databases and queries described in DESIGN.md §"Input recipe".  Both `oracle/`
and `paper_1404_4152_b200/` consumers read the same bytes from here.
"""
from .alphabet import ALPHABET, DUMMY, encode, decode  # noqa: F401
from .matrices import blosum62, blosum50, matrix32  # noqa: F401
from .synth import (CONFIGS, SynthDB, make_db, make_query, gen_residues, random_db, db_lengths,  # noqa: F401
                    lognormal_lengths, splitmix64, stream_key, uniform_u64, manifest_hash)
