"""pytest plugin: run the reference's OWN test suite against this engine.

Loaded with ``-p mbu_conformance`` into a pytest run over
``baseline/_ref/bitunet_tests`` (the unmodified ``bitunet`` 0.1.0 tests,
installed by ``tools/install_reference.sh``). Before the test modules are
collected it rebinds ``bitunet``'s compute functions to the GPU engine
through ``paper_2601_11660_b200.plug.install`` — the reference's own plug
point (``graph.forward`` dispatches through module-level names,
``pkg/src/bitunet/graph.py:434-451``) — so every ``from bitunet.layers import
conv_forward`` in those tests gets the GPU op. ``MBU_PLUG`` selects what is
rebound: ``layers`` (the layer functions; the reference's interpreter loop
drives them), ``forward`` (the whole-network native forward) or ``all``.
"""

from __future__ import annotations

import os


def pytest_configure(config):
    import bitunet

    import paper_2601_11660_b200 as mb
    from paper_2601_11660_b200 import plug

    level = os.environ.get("MBU_PLUG", "all")
    restore = plug.install(bitunet, layers=level in ("all", "layers"),
                           forward=level in ("all", "forward"))
    config._mbu_restore = restore
    # the engine's errors must BE the reference's (the suite catches bitunet.errors.*)
    assert issubclass(mb.ShapeError, bitunet.errors.ShapeError), "reference error aliasing inactive"
    names = sorted({f"{m}.{a}" for m, a in restore.rebound})
    print(f"\nmbu_conformance: MBU_PLUG={level}, {len(names)} bindings rebound to the GPU engine")


def pytest_report_header(config):
    r = getattr(config, "_mbu_restore", None)
    if r is None:
        return None
    return "mbu_conformance rebound: " + ", ".join(sorted({f"{m}.{a}" for m, a in r.rebound}))


def pytest_unconfigure(config):
    r = getattr(config, "_mbu_restore", None)
    if r is not None:
        r()
