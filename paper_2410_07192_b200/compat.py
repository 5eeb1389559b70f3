"""Expose this package under the reference's module names (``bubblefill.*``).

``install()`` registers ``bubblefill``, ``bubblefill.pipeline``, ``.workload``,
``.partition``, ``.coordinator``, ``.placer`` and ``.sim`` in ``sys.modules`` as
aliases of this package's modules, so code (and the reference's own test-suite)
written against ``bubblefill`` runs unchanged on the B200 build. The reference's
INI config loader and CLI are out of scope.
"""

from __future__ import annotations

import importlib
import sys
import types

ALIASES = {
    "pipeline": "schedule",
    "workload": "profiles",
    "partition": "planner",
    "coordinator": "coordinator",
    "placer": "routing",
    "sim": "sim",
}


def install(name: str = "bubblefill") -> types.ModuleType:
    root = importlib.import_module(__package__)
    pkg = types.ModuleType(name)
    pkg.__path__ = []  # mark as a package
    pkg.__dict__.update({k: v for k, v in vars(root).items() if not k.startswith("__")})
    pkg.__version__ = root.__version__
    sys.modules[name] = pkg
    for ref_name, ours in ALIASES.items():
        mod = importlib.import_module(f"{__package__}.{ours}")
        sys.modules[f"{name}.{ref_name}"] = mod
        setattr(pkg, ref_name, mod)
    return pkg
