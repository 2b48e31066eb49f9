"""The oracle's pins, run again inside the GPU session.

`pytest -m gpu` is what the driver runs on the GPU box; the CPU tests that
pin the C restatement (oracle/fde_oracle.c) to the reference's golden vectors
and to the unmodified reference build (oracle/_ref, which travels with the
snapshot) are deselected there.  This module re-runs them under the gpu
marker, so the checker the parity tests trust is itself checked in the same
driver-run session, on the same box."""
import inspect

import pytest

import test_oracle_pins as pins
import test_unpinned_rows as unpinned

pytestmark = pytest.mark.gpu


def _cases(mod):
    for name, fn in sorted(vars(mod).items()):
        if name.startswith("test_") and callable(fn):
            yield name, fn


def _param_sets(fn):
    """Expand the function's own @pytest.mark.parametrize marks."""
    sets = [{}]
    for mark in getattr(fn, "pytestmark", []):
        if mark.name != "parametrize":
            continue
        names = [a.strip() for a in mark.args[0].split(",")] if isinstance(mark.args[0], str) \
            else list(mark.args[0])
        new = []
        for base in sets:
            for vals in mark.args[1]:
                vals = vals if isinstance(vals, (tuple, list)) and len(names) > 1 else (vals,)
                new.append(dict(base, **dict(zip(names, vals))))
        sets = new
    return sets


@pytest.mark.parametrize("name", [n for n, _ in _cases(pins)])
def test_oracle_pin(name, orc, request):
    fn = getattr(pins, name)
    want = inspect.signature(fn).parameters
    fixtures = {"orc": orc}
    if "ref" in want:
        fixtures["ref"] = request.getfixturevalue("ref")
    for params in _param_sets(fn):
        fn(**{k: v for k, v in {**fixtures, **params}.items() if k in want})


@pytest.mark.parametrize("name", ["test_wsgd_1m1_hand_values",
                                  "test_wsgd_lambda_formula_reproduces_both_tables",
                                  "test_wsgd_second_order_on_manufactured_solution"])
def test_unpinned_row_pin(name, orc):
    fn = getattr(unpinned, name)
    want = inspect.signature(fn).parameters
    for params in _param_sets(fn):
        fn(**{k: v for k, v in {"orc": orc, **params}.items() if k in want})
