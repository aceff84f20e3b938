"""pytest plugin: make `import binfec...` resolve to this repo's GPU shim.

Used by tests/test_reference_suite.py to re-run the reference's OWN test
suite (staged by tools/stage_reference.sh into the git-ignored
baseline/_ref/ref_tests) against the drop-in (SURVEY §8b "parity harness
through the boundary").  Loaded with `-p binfec_shim_plugin`, i.e. before the
reference's conftest.py imports binfec.

* binfec.{field, transform, derivative, walsh, rs, batch} are the shim's
  modules themselves: every compute call goes through liblch.so.
* binfec.basis is the shim's module with one addition: the reference's TEST
  oracles `eval_x_naive` / `eval_poly_naive` (basis.py:111-132; the product
  does not carry them) are delegated to the unmodified reference, loaded
  under the name `binfec_ref` from baseline/_ref.
"""

from __future__ import annotations

import importlib.util
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "baseline", "_ref", "binfec")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _load_reference():
    spec = importlib.util.spec_from_file_location(
        "binfec_ref", os.path.join(REF, "__init__.py"), submodule_search_locations=[REF])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["binfec_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def _install() -> None:
    ref = _load_reference()
    ref_basis = importlib.import_module("binfec_ref.basis")
    ref_field = importlib.import_module("binfec_ref.field")

    import paper_1404_3458_b200 as shim
    from paper_1404_3458_b200 import basis, batch, derivative, field, rs, transform, walsh

    class BasisTables(basis.BasisTables):
        """The shim's tables + the reference's naive evaluators (test oracles)."""

        _ref_bt = None

        def _ref(self):
            if self._ref_bt is None:
                p = self.ft.params
                rft = ref_field.tables_for(p.r, p.reduction_poly)
                self._ref_bt = ref_basis.build_basis_tables(rft, self.max_h)
            return self._ref_bt

        def eval_x_naive(self, i, x):
            return self._ref().eval_x_naive(i, x)

        def eval_poly_naive(self, coeffs, x):
            return self._ref().eval_poly_naive(coeffs, x)

    basis_mod = types.ModuleType("binfec.basis")
    basis_mod.__dict__.update({k: v for k, v in vars(basis).items() if not k.startswith("__")})
    basis_mod.BasisTables = BasisTables
    basis_mod.build_basis_tables = lambda ft, max_h: BasisTables(ft, max_h)

    pkg = types.ModuleType("binfec")
    pkg.__path__ = []
    pkg.__dict__.update({k: v for k, v in vars(shim).items() if not k.startswith("__")})
    pkg.build_basis_tables = basis_mod.build_basis_tables
    pkg.BasisTables = BasisTables
    mods = {"field": field, "basis": basis_mod, "transform": transform, "derivative": derivative,
            "walsh": walsh, "rs": rs, "batch": batch}
    sys.modules["binfec"] = pkg
    for name, mod in mods.items():
        sys.modules["binfec." + name] = mod
        setattr(pkg, name, mod)
    pkg.__shim_of__ = ref.__name__


_install()


def pytest_report_header(config):
    return "binfec -> paper_1404_3458_b200 (GPU shim); test oracles from baseline/_ref"
