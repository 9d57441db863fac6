"""Exception types of the drop-in (``rts_sph.errors``, errors.py:4-10).

Same class hierarchy as the reference so ``except`` clauses keep working:
``ConfigError`` is a ``ValueError``; ``NumericalError`` a ``RuntimeError``.
The B200 kernels never raise; they set bits in a device error word which the
host reads once per step (per minor step for PCISPH) and turns into these.
"""


class ConfigError(ValueError):
    """Invalid scene text, preset, schedule or solver configuration."""


class NumericalError(RuntimeError):
    """The run left its stable regime: escaped or non-finite particles, a
    collapsed neighbourhood, or a pressure solve that hit its iteration cap."""
