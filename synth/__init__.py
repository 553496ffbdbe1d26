"""Seeded synthetic STA workloads shared by the CUDA path and the oracle.

This package holds ONLY input generators: netlists, NLDM table pools, RC trees
and constraints as flat arrays.  It contains none of the timing arithmetic
(no LUT evaluation, no Elmore, no propagation) -- see DESIGN.md §3 "input
recipe".  Both `oracle/` (test infrastructure) and the product binding consume
the same `Design` objects.
"""
from .design import (  # noqa: F401
    Design, Library, RcTree, Constraints, Logic, CaseValues, truth_table,
    SENSE_POS, SENSE_NEG, SENSE_NON, SENSE_RISE_EDGE, SENSE_FALL_EDGE,
    ROLE_INTERNAL, ROLE_PI, ROLE_PO, ROLE_FF_CK, ROLE_FF_D, NO_PIN,
)
from .hand import c17, h1_chain, h3_reg2reg, h4_seeds  # noqa: F401
from .recipe import generate, CONFIGS, config_design, corner_scales  # noqa: F401
from .place import placement, UNITS as STEINER_UNITS  # noqa: F401
