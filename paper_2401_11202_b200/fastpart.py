"""Indexed value lookups for the reference partitioner.

The reference's rewrite engine answers "where is %x defined" (`ir.find_def`,
ir.py:452-471) and "who uses %x" (`ir.collect_uses`, ir.py:487-505) with a
linear walk over the whole function, and `_propagate_once`/`_match_site`
(rewrite.py:285-376) ask these questions for every op on every propagation
pass: O(ops^2) per tactic.  Profiled on a 2-block transformer BP+MP, the two
walks are 78% of partitioning time; a 32-block C3 partition takes ~2 h.

`fast_partitioning()` answers the same questions from a per-function index
(definitions and use lists in the reference's traversal order, so results are
identical, including list order) that is rebuilt lazily after any mutation:
the functions that mutate the IR during propagation (`apply_tile`,
`apply_atomic`, `_rewrite_site`, `_fuse_once`, `replace_uses`,
rewrite.py:189-420, ir.py:508) do all their lookups before they mutate, so
they are wrapped to invalidate the index when they return; the SPMD lowering
that `Partitioner.costs` runs after each tactic (`lower_to_spmd`, `localize`,
spmd.py:212-261) interleaves lookups with in-place rewrites, so inside it
lookups fall back to the reference's own walks.  Nothing in the reference is edited;
the patch is installed for the duration of the context only.

    from paper_2401_11202_b200.fastpart import fast_partitioning
    with fast_partitioning():
        for t in schedule: partitioner.apply(t)

`verify=True` (or SPX_FASTPART_VERIFY=1) runs both implementations on every
query and raises on any difference (used by the tests).
"""
from __future__ import annotations

import contextlib
import os
import sys

__all__ = ["fast_partitioning"]

# Rewrites that do all their lookups first and mutate last (then return):
# the index stays valid for their queries and is invalidated when they return.
_MUTATE_LAST = {"rewrite": ["apply_tile", "apply_atomic", "_rewrite_site", "_fuse_once", "replace_uses"],
                "ir": ["replace_uses"]}
# SPMD lowering (run by Partitioner.costs after every tactic) interleaves
# lookups with in-place rewrites of its copy: reference walks inside.
_MUTATE_INTERLEAVED = {"spmd": ["lower_to_spmd", "localize"]}


class _Index:
    """Definitions and uses of every value of one function, in the reference's
    traversal order (pre-order over ops; an op's results before its regions;
    a region's argument before the region's ops; region ops before yields)."""

    def __init__(self, func):
        self.args = {}
        for i, (n, _) in enumerate(func.args):
            self.args.setdefault(n, i)
        self.defs = {}
        self.uses = {}
        self._walk(func.ops, ())
        self.results = {}
        for j, r in enumerate(func.results):
            self.results.setdefault(r, []).append(j)

    def _walk(self, ops, axes):
        defs, uses = self.defs, self.uses
        for i, op in enumerate(ops):
            for ri, r in enumerate(op.results):
                defs.setdefault(r, (ops, i, op, ri, axes))
            for j, o in enumerate(op.operands):
                uses.setdefault(o, []).append(("op", op, j))
            for region in op.regions:
                defs.setdefault(region.arg, ("rangearg", op, region, axes))
                inner = axes + ((op.attrs["axis"],) if op.kind == "loop" else ())
                self._walk(region.ops, inner)
                for j, y in enumerate(region.yields):
                    uses.setdefault(y, []).append(("yield", op, region, j))


class _State:
    def __init__(self, orig_find_def, orig_collect_uses, verify):
        self.gen = 0
        self.depth = 0
        self.cache = {}        # id(func) -> (gen, func, index)
        self.orig_find_def = orig_find_def
        self.orig_collect_uses = orig_collect_uses
        self.verify = verify
        self.hits = 0
        self.rebuilds = 0

    def index(self, func):
        ent = self.cache.get(id(func))
        if ent is not None and ent[0] == self.gen and ent[1] is func:
            self.hits += 1
            return ent[2]
        idx = _Index(func)
        self.rebuilds += 1
        self.cache[id(func)] = (self.gen, func, idx)
        return idx


def _make(state):
    def find_def(func, name):
        if state.depth:
            return state.orig_find_def(func, name)
        idx = state.index(func)
        if name in idx.args:
            got = ("arg", idx.args[name])
        elif name in idx.defs:
            got = idx.defs[name]
        else:
            got = None
        if state.verify:
            try:
                want = state.orig_find_def(func, name)
            except KeyError:
                want = None
            same = (got is None and want is None) or (
                got is not None and want is not None and len(got) == len(want)
                and all(a is b or a == b for a, b in zip(got, want)))
            if not same:
                raise AssertionError(f"fastpart: find_def(%{name}) differs: {got!r} vs {want!r}")
        if got is None:
            raise KeyError(f"value %{name} not defined in @{func.name}")
        return got

    def collect_uses(func, name):
        if state.depth:
            return state.orig_collect_uses(func, name)
        idx = state.index(func)
        out = list(idx.uses.get(name, ()))
        out.extend(("return", j) for j in idx.results.get(name, ()))
        if state.verify:
            want = state.orig_collect_uses(func, name)
            if len(out) != len(want) or any(
                    len(a) != len(b) or any(x is not y and x != y for x, y in zip(a, b))
                    for a, b in zip(out, want)):
                raise AssertionError(f"fastpart: collect_uses(%{name}) differs")
        return out

    return find_def, collect_uses


def _mutating(state, fn, interleaved):
    def wrapper(*a, **kw):
        state.gen += 1
        if interleaved:
            state.depth += 1
        try:
            return fn(*a, **kw)
        finally:
            if interleaved:
                state.depth -= 1
            state.gen += 1
    wrapper.__wrapped__ = fn
    return wrapper


@contextlib.contextmanager
def fast_partitioning(verify: bool | None = None):
    """Install the indexed lookups into the reference's modules (spindle.ir,
    spindle.rewrite and every spindle module that imported them by name)."""
    from spindle import ir, rewrite, spmd   # the reference package (must be importable)
    if verify is None:
        verify = os.environ.get("SPX_FASTPART_VERIFY", "0") == "1"
    state = _State(ir.find_def, ir.collect_uses, verify)
    find_def, collect_uses = _make(state)
    saved = []
    mods = [m for n, m in sys.modules.items() if n == "spindle" or n.startswith("spindle.")]

    def patch(name, new, orig):
        for m in mods:
            if getattr(m, name, None) is orig:
                saved.append((m, name, orig))
                setattr(m, name, new)

    patch("find_def", find_def, state.orig_find_def)
    patch("collect_uses", collect_uses, state.orig_collect_uses)
    for table, interleaved in ((_MUTATE_LAST, False), (_MUTATE_INTERLEAVED, True)):
        for modname, names in table.items():
            mod = {"ir": ir, "rewrite": rewrite, "spmd": spmd}[modname]
            for n in names:
                orig = getattr(mod, n)
                if getattr(orig, "__wrapped__", None) is not None:
                    continue
                patch(n, _mutating(state, orig, interleaved), orig)
    try:
        yield state
    finally:
        for m, name, orig in reversed(saved):
            setattr(m, name, orig)
