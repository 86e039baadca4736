"""Drop-in alias: ``import chunkstar`` resolves to paper_2108_05818_b200.

Put ``<repo>/dropin`` first on ``PYTHONPATH`` and the reference's own
hot-path tests (`/root/reference/pkg/tests`) import this build's modules
under their original names (``chunkstar.fsm``, ``chunkstar.engine`` …).
The package's search path is redirected to the real package directory,
so every ``chunkstar.X`` is the module ``paper_2108_05818_b200/X.py``.
"""

import os as _os

__path__ = [_os.path.join(_os.path.dirname(_os.path.dirname(
    _os.path.dirname(_os.path.abspath(__file__)))), "paper_2108_05818_b200")]

with open(_os.path.join(__path__[0], "__init__.py")) as _f:
    exec(compile(_f.read(), __path__[0] + "/__init__.py", "exec"))
