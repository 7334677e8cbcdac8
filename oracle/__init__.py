"""TEST INFRASTRUCTURE ONLY: CPU parity checkers (see oracle/checkers.py).

Importable only by tests/, __graft_entry__.smoke() and bench.py's CPU
baseline legs; the product package never imports it.
"""
from .checkers import (ORACLE_SO, REF_SO, Oracle, RefError, Reference, bf16_to_f64, build,
                       f32_to_bf16_bits, model_from_reference_layout)

__all__ = ["ORACLE_SO", "REF_SO", "Oracle", "RefError", "Reference", "bf16_to_f64", "build",
           "f32_to_bf16_bits", "model_from_reference_layout"]
