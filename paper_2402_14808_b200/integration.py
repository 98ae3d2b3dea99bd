"""Install the B200 relay path into the reference package `relayserve`.

The reference's kernel switch (`relayserve/kernels.py:14-37`) selects a
per-head float64 backend and re-exports five functions from it; the B200
path works one level up, per attention segment, so it is wired in at the
operator API instead (`relayserve/attention.py`), leaving `kernels.py` and
its five re-exports untouched.

`install()` rebinds, in the live reference modules:

  relayserve.attention  naive_causal_attention (attention.py:72), attention_with_lse (:96),
                        relay_fusion (:137), relay_attention_ragged (:203),
                        relay_attention (:246), baseline_attention_ragged (:266),
                        baseline_attention (:291)
  relayserve.model      the names model.py:24-26 imported by value:
                        attention_with_lse, baseline_attention_ragged, relay_attention_ragged

so the reference's own callers -- `DecoderModel._attend` (model.py:314-336),
the CLI and the tests -- run on librelay_b200.so.  Errors keep the
reference's types: this package's DimensionError / ContractError are
re-raised as relayserve.errors.DimensionError / ContractError.  `uninstall()`
restores the originals.  INTEGRATION.md shows the equivalent edit a
maintainer would make inside attention.py.
"""

from __future__ import annotations

import functools
import importlib

from . import attention as _b200
from . import errors as _errors

ATTENTION_NAMES = ("naive_causal_attention", "attention_with_lse", "relay_fusion",
                   "relay_attention_ragged", "relay_attention", "baseline_attention_ragged",
                   "baseline_attention")
MODEL_NAMES = ("attention_with_lse", "baseline_attention_ragged", "relay_attention_ragged")

_saved: dict = {}


def _reraise_as(ref_errors, fn):
    mapping = ((_errors.DimensionError, ref_errors.DimensionError),
               (_errors.ContractError, ref_errors.ContractError),
               (_errors.NonFiniteError, ref_errors.NonFiniteError))

    @functools.wraps(fn)
    def wrapped(*args, **kwargs):
        try:
            return fn(*args, **kwargs)
        except tuple(ours for ours, _ in mapping) as exc:
            for ours, theirs in mapping:
                if isinstance(exc, ours):
                    raise theirs(str(exc)) from exc
            raise
    wrapped.__b200__ = True
    return wrapped


def install(package: str = "relayserve"):
    """Route `package`'s attention entry points (and the model's imported
    names) to the B200 kernels.  Idempotent; returns the patched modules."""
    att = importlib.import_module(f"{package}.attention")
    ref_errors = importlib.import_module(f"{package}.errors")
    try:
        model = importlib.import_module(f"{package}.model")
    except ImportError:
        model = None
    targets = [(att, ATTENTION_NAMES)] + ([(model, MODEL_NAMES)] if model is not None else [])
    for mod, names in targets:
        for name in names:
            cur = getattr(mod, name)
            if getattr(cur, "__b200__", False):
                continue
            _saved[(mod.__name__, name)] = cur
            setattr(mod, name, _reraise_as(ref_errors, getattr(_b200, name)))
    return [mod for mod, _ in targets]


def uninstall():
    """Restore every function `install` replaced."""
    import sys
    for (modname, name), fn in list(_saved.items()):
        mod = sys.modules.get(modname)
        if mod is not None:
            setattr(mod, name, fn)
    _saved.clear()
