"""The documented binding (paper_2402_14808_b200.integration)
applied to the reference modules compiled from /root/reference into
oracle/_ref (CPU part: wiring only, no kernel calls).

* `relayserve.kernels` still imports with its five re-exports
  (kernels.py:33-37) -- the B200 path is not a kernels.py backend.
* install() rebinds relayserve.attention's operator API and the names
  model.py:24-26 imported by value; uninstall() restores them.
"""

import os
import sys

import pytest

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


@pytest.fixture()
def relayserve():
    if not os.path.isdir(os.path.join(REF, "relayserve")):
        pytest.skip("oracle/_ref not built (python oracle/build.py)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import relayserve.attention  # noqa: F401
    import relayserve.kernels
    import relayserve.model  # noqa: F401
    return sys.modules["relayserve"]


def test_kernels_module_untouched(relayserve):
    from paper_2402_14808_b200 import integration
    integration.install()
    try:
        k = sys.modules["relayserve.kernels"]
        for name in ("matmul_nt", "softmax_lse_rows", "softmax_lse_prefix", "rope_rows",
                     "naive_attention_head"):
            assert callable(getattr(k, name))
        assert k.BACKEND in ("compiled", "pure-python")
    finally:
        integration.uninstall()


def test_install_rebinds_attention_and_model(relayserve):
    from paper_2402_14808_b200 import attention as b200
    from paper_2402_14808_b200 import integration
    att = sys.modules["relayserve.attention"]
    model = sys.modules["relayserve.model"]
    before = {n: getattr(att, n) for n in integration.ATTENTION_NAMES}
    before_m = {n: getattr(model, n) for n in integration.MODEL_NAMES}
    integration.install()
    integration.install()   # idempotent
    try:
        for n in integration.ATTENTION_NAMES:
            assert getattr(att, n).__wrapped__ is getattr(b200, n)
        for n in integration.MODEL_NAMES:
            assert getattr(model, n).__wrapped__ is getattr(b200, n)
        # errors surface as the reference's own types
        import numpy as np
        from relayserve.errors import ContractError
        with pytest.raises(ContractError):
            att.relay_attention(np.zeros((1, 1, 1, 2)), np.zeros((0, 1, 2)), np.zeros((0, 1, 2)),
                                [np.zeros((1, 1, 2))], [np.zeros((1, 1, 2))])
    finally:
        integration.uninstall()
    assert all(getattr(att, n) is f for n, f in before.items())
    assert all(getattr(model, n) is f for n, f in before_m.items())
