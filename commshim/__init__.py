"""Drop-in alias: ``import commshim`` resolves to :mod:`paper_2101_08878_b200`.

Code written against the reference package (``pkg/src/commshim``) imports
``commshim``, ``commshim.transport``, ``commshim.messaging`` … unchanged; every
such module is the *same object* as its ``paper_2101_08878_b200`` counterpart
(no duplicate classes, so ``isinstance`` and ``except`` clauses agree).
"""

from __future__ import annotations

import importlib
import importlib.abc
import importlib.util
import sys

_REAL = "paper_2101_08878_b200"
_ALIAS = __name__  # "commshim"


class _AliasLoader(importlib.abc.MetaPathFinder, importlib.abc.Loader):
    def find_spec(self, fullname, path=None, target=None):
        if fullname.startswith(_ALIAS + "."):
            real = _REAL + fullname[len(_ALIAS):]
            if importlib.util.find_spec(real) is None:
                return None
            return importlib.util.spec_from_loader(fullname, self, is_package=True)
        return None

    _specs: dict = {}

    def create_module(self, spec):
        module = importlib.import_module(_REAL + spec.name[len(_ALIAS):])
        self._specs[id(module)] = module.__spec__
        return module

    def exec_module(self, module):
        # importlib stamped the alias spec onto the real module; put the real one back.
        module.__spec__ = self._specs.pop(id(module), module.__spec__)


if not any(isinstance(f, _AliasLoader) for f in sys.meta_path):
    sys.meta_path.insert(0, _AliasLoader())

_real_pkg = importlib.import_module(_REAL)
sys.modules[_ALIAS] = _real_pkg
