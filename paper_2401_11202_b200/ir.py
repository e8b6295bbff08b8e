"""Read-only data model for localized SPMD programs.

The backend consumes the reference's *localized* modules (the output of
`localize(lower_to_spmd(...))`, /root/reference/pkg/src/spindle/spmd.py:212-261):
straight-line functions over a named mesh whose ops are the eleven tensor op
kinds plus the five collectives (`ir.py:18-24`).  The reference package is not
present on the GPU box, so this module restates the part of its data model the
evaluator reads -- with the same attribute names, so reference `Module`
objects and ours are interchangeable at the `spmd_interpret` boundary
(duck-typed):

  TensorType.dims/.elem          ir.py:31-59
  Mesh.axes/.names()/.size()/.coords()   ir.py:70-128 (coords row-major, first
                                 axis slowest, ir.py:103-108)
  Op.kind/.results/.result_types/.operands/.attrs   ir.py:180-197
  Func.name/.args/.ops/.results/.result_types       ir.py:200-215
  Module.funcs/.mesh/.func()     ir.py:218-230
  ShardingSpec.args/.results     spmd.py:45-57

`parse_module` reads the canonical text form (`printer.py:41-104`) for the
straight-line subset (everything a localized or dense module can contain; no
partitioning loops).  Shapes are re-derived with the reference's shape rules
(`ir.py:240-393`) so a malformed cached program fails at load, not on device.
"""
from __future__ import annotations

import json
import re
from dataclasses import dataclass, field

ELEM_KINDS = ("f32", "i32")
TENSOR_OP_KINDS = ("constant", "matmul", "add", "mul", "neg", "exp",
                   "transpose", "reduce", "reshape", "broadcast", "tag")
COLLECTIVE_KINDS = ("all_slice", "all_gather", "all_reduce", "reduce_scatter", "all_to_all")
COUNTED_COLLECTIVES = ("all_gather", "all_reduce", "reduce_scatter", "all_to_all")


class ShapeError(Exception):
    pass


class ParseError(Exception):
    pass


def _prod(xs) -> int:
    n = 1
    for x in xs:
        n *= int(x)
    return n


@dataclass(frozen=True)
class TensorType:
    dims: tuple
    elem: str = "f32"

    @property
    def rank(self) -> int:
        return len(self.dims)

    @property
    def elems(self) -> int:
        return _prod(self.dims)

    @property
    def nbytes(self) -> int:
        return 4 * self.elems

    def render(self) -> str:
        return "tensor<" + "x".join([str(d) for d in self.dims] + [self.elem]) + ">"


@dataclass(frozen=True)
class Mesh:
    axes: tuple

    def names(self):
        return [n for n, _ in self.axes]

    def size(self, name: str) -> int:
        for n, s in self.axes:
            if n == name:
                return s
        raise KeyError(f"no mesh axis named {name!r}")

    @property
    def device_count(self) -> int:
        return _prod(s for _, s in self.axes)

    def coords(self):
        out = [dict()]
        for name, size in self.axes:
            out = [{**c, name: i} for c in out for i in range(size)]
        return out

    @staticmethod
    def parse(text: str) -> "Mesh":
        axes = []
        for part in text.strip().strip("{}").split(","):
            part = part.strip()
            if not part:
                continue
            m = re.fullmatch(r"([A-Za-z_]\w*)\s*:\s*(\d+)", part)
            if not m:
                raise ValueError(f"bad mesh axis {part!r}")
            axes.append((m.group(1), int(m.group(2))))
        return Mesh(tuple(axes))


@dataclass
class Op:
    kind: str
    results: list
    result_types: list
    operands: list
    attrs: dict = field(default_factory=dict)
    regions: list = field(default_factory=list)

    @property
    def result(self) -> str:
        return self.results[0]

    @property
    def result_type(self) -> TensorType:
        return self.result_types[0]


@dataclass
class Func:
    name: str
    args: list
    ops: list
    results: list
    result_types: list

    def arg_names(self):
        return [n for n, _ in self.args]


@dataclass
class Module:
    funcs: list
    mesh: Mesh | None = None

    def func(self, name: str = "main") -> Func:
        for f in self.funcs:
            if f.name == name:
                return f
        raise KeyError(f"no function named {name!r}")


@dataclass
class ShardingSpec:
    args: dict = field(default_factory=dict)
    results: list = field(default_factory=list)

    def to_json(self) -> dict:
        return {"args": self.args, "results": self.results}

    @staticmethod
    def from_json(d) -> "ShardingSpec":
        if isinstance(d, str):
            d = json.loads(d)
        return ShardingSpec(dict(d["args"]), list(d["results"]))


# --- shape rules (restated from ir.py:240-393, straight-line subset) --------

def _need(cond, msg):
    if not cond:
        raise ShapeError(msg)


def _axes_n(axes, mesh) -> int:
    return _prod(mesh.size(a) for a in axes)


def infer_result_type(kind: str, ts: list, attrs: dict, mesh) -> TensorType:
    if kind == "constant":
        return attrs["type"]
    if kind == "matmul":
        a, b = ts
        _need(a.rank == 2 and b.rank == 2 and a.dims[1] == b.dims[0],
              f"matmul {a.dims} @ {b.dims}")
        return TensorType((a.dims[0], b.dims[1]), a.elem)
    if kind in ("add", "mul"):
        _need(ts[0] == ts[1], f"{kind} operand mismatch {ts[0]} vs {ts[1]}")
        return ts[0]
    if kind in ("neg", "exp", "tag", "all_reduce"):
        return ts[0]
    a = ts[0]
    if kind == "transpose":
        perm = attrs["perm"]
        _need(sorted(perm) == list(range(a.rank)), f"bad perm {perm}")
        return TensorType(tuple(a.dims[p] for p in perm), a.elem)
    if kind == "reduce":
        dims = attrs["dims"]
        _need(len(dims) > 0 and all(0 <= d < a.rank for d in dims), f"bad reduce dims {dims}")
        return TensorType(tuple(d for i, d in enumerate(a.dims) if i not in dims), a.elem)
    if kind == "reshape":
        dims = tuple(attrs["dims"])
        _need(_prod(dims) == a.elems, f"reshape {a.dims} -> {dims}")
        return TensorType(dims, a.elem)
    if kind == "broadcast":
        shape, dims = tuple(attrs["shape"]), list(attrs["dims"])
        _need(len(dims) == a.rank and all(shape[d] == a.dims[i] for i, d in enumerate(dims)),
              f"bad broadcast {a.dims} -> {shape} via {dims}")
        return TensorType(shape, a.elem)
    if kind in ("all_slice", "reduce_scatter"):
        nd = list(a.dims)
        for d, axes in enumerate(attrs["axes_per_dim"]):
            n = _axes_n(axes, mesh)
            _need(nd[d] % n == 0, f"{kind} dim {d} of {a.dims} not divisible by {n}")
            nd[d] //= n
        return TensorType(tuple(nd), a.elem)
    if kind == "all_gather":
        nd = list(a.dims)
        for d, axes in enumerate(attrs["axes_per_dim"]):
            nd[d] *= _axes_n(axes, mesh)
        return TensorType(tuple(nd), a.elem)
    if kind == "all_to_all":
        n = _axes_n(attrs["axes"], mesh)
        gd, sd = attrs["gather_dim"], attrs["slice_dim"]
        nd = list(a.dims)
        _need(nd[sd] % n == 0, "all_to_all slice dim not divisible")
        nd[gd] *= n
        nd[sd] //= n
        return TensorType(tuple(nd), a.elem)
    raise ShapeError(f"unknown op kind {kind!r}")


# --- text parser (canonical form of printer.py:41-104) ----------------------

_TOK = re.compile(r"""
    (?P<ws>\s+|//[^\n]*)
  | (?P<ttype>tensor<[^<>]*>)
  | (?P<arrow>->)
  | (?P<num>-?(?:\d+\.?\d*(?:[eE][+-]?\d+)?|inf|nan))
  | (?P<var>%[A-Za-z0-9_.]+)
  | (?P<str>"[^"\n]*")
  | (?P<ident>[A-Za-z_]\w*)
  | (?P<p>[(){}\[\],:=@<>])
""", re.VERBOSE)


class _Toks:
    def __init__(self, text: str):
        self.t = []
        pos = 0
        while pos < len(text):
            m = _TOK.match(text, pos)
            if not m:
                raise ParseError(f"unexpected {text[pos:pos + 20]!r}")
            if m.lastgroup != "ws":
                self.t.append((m.lastgroup, m.group()))
            pos = m.end()
        self.t.append(("eof", ""))
        self.i = 0

    def peek(self, k=0):
        return self.t[min(self.i + k, len(self.t) - 1)]

    def next(self):
        tok = self.t[self.i]
        self.i += 1
        return tok

    def expect(self, kind, text=None):
        tok = self.next()
        if tok[0] != kind or (text is not None and tok[1] != text):
            raise ParseError(f"expected {text or kind!r}, got {tok[1]!r}")
        return tok[1]

    def accept(self, kind, text=None):
        tok = self.peek()
        if tok[0] == kind and (text is None or tok[1] == text):
            self.i += 1
            return tok[1]
        return None


def _ttype(tk: _Toks) -> TensorType:
    body = tk.expect("ttype")[len("tensor<"):-1].split("x")
    if body[-1] not in ELEM_KINDS:
        raise ParseError(f"bad element kind {body[-1]!r}")
    return TensorType(tuple(int(p) for p in body[:-1]), body[-1])


def _var(tk):
    return tk.expect("var")[1:]


def _strlist(tk):
    tk.expect("p", "[")
    out = []
    while not tk.accept("p", "]"):
        if out:
            tk.expect("p", ",")
        out.append(tk.expect("str")[1:-1])
    return out


def _apd(tk):
    tk.expect("p", "[")
    out = []
    while not tk.accept("p", "]"):
        if out:
            tk.expect("p", ",")
        out.append(_strlist(tk))
    return out


def _monoid(tk):
    if tk.accept("p", "<"):
        m = tk.expect("ident")
        tk.expect("p", ">")
        return m
    return "sum"


def _braces(tk) -> dict:
    attrs = {}
    if not tk.accept("p", "{"):
        return attrs
    while not tk.accept("p", "}"):
        if attrs:
            tk.expect("p", ",")
        key = tk.expect("ident")
        tk.expect("p", "=")
        if tk.accept("p", "["):
            vals = []
            while not tk.accept("p", "]"):
                if vals:
                    tk.expect("p", ",")
                vals.append(int(tk.expect("num")))
            attrs[key] = vals
        elif tk.peek()[0] == "ident":
            attrs[key] = tk.next()[1]
        else:
            attrs[key] = int(tk.expect("num"))
    return attrs


def _op(tk: _Toks, types: dict, mesh) -> Op:
    results = [_var(tk)]
    while tk.accept("p", ","):
        results.append(_var(tk))
    tk.expect("p", "=")
    kind = tk.expect("ident")
    attrs: dict = {}
    operands: list = []

    def operand():
        n = _var(tk)
        if n not in types:
            raise ParseError(f"use of undefined value %{n}")
        operands.append(n)

    if kind == "constant":
        attrs["value"] = float(tk.expect("num"))
    elif kind in ("matmul", "add", "mul"):
        operand()
        tk.expect("p", ",")
        operand()
    elif kind in ("neg", "exp"):
        operand()
    elif kind in ("transpose", "reduce", "reshape", "broadcast"):
        operand()
        attrs.update(_braces(tk))
        if kind == "reduce":
            attrs.setdefault("monoid", "sum")
    elif kind == "tag":
        attrs["name"] = tk.expect("str")[1:-1]
        operand()
    elif kind == "all_reduce":
        attrs["monoid"] = _monoid(tk)
        attrs["axes"] = _strlist(tk)
        operand()
    elif kind in ("all_slice", "all_gather"):
        attrs["axes_per_dim"] = _apd(tk)
        operand()
    elif kind == "all_to_all":
        attrs["gather_dim"] = int(tk.expect("num"))
        tk.expect("arrow")
        attrs["slice_dim"] = int(tk.expect("num"))
        attrs["axes"] = _strlist(tk)
        operand()
    elif kind == "reduce_scatter":
        attrs["monoid"] = _monoid(tk)
        attrs["axes"] = _strlist(tk)
        attrs["axes_per_dim"] = _apd(tk)
        operand()
    else:
        raise ParseError(f"op kind {kind!r} is not part of a straight-line program")
    tk.expect("p", ":")
    declared = _ttype(tk)
    if kind == "constant":
        attrs["type"] = declared
    if kind == "broadcast":
        attrs["shape"] = list(declared.dims)
    inferred = infer_result_type(kind, [types[o] for o in operands], attrs, mesh)
    if inferred != declared:
        raise ParseError(f"%{results[0]}: declared {declared.render()}, rules give {inferred.render()}")
    for r in results:
        if r in types:
            raise ParseError(f"redefinition of %{r}")
        types[r] = declared
    return Op(kind, results, [declared], operands, attrs)


def parse_module(text: str) -> Module:
    tk = _Toks(text)
    mesh = None
    if tk.accept("ident", "mesh"):
        tk.expect("p", "{")
        axes = []
        while not tk.accept("p", "}"):
            if axes:
                tk.expect("p", ",")
            name = tk.expect("ident")
            tk.expect("p", ":")
            axes.append((name, int(tk.expect("num"))))
        mesh = Mesh(tuple(axes))
    funcs = []
    while tk.peek()[0] != "eof":
        tk.expect("ident", "func")
        tk.expect("p", "@")
        fname = tk.expect("ident")
        tk.expect("p", "(")
        args, types = [], {}
        while not tk.accept("p", ")"):
            if args:
                tk.expect("p", ",")
            n = _var(tk)
            tk.expect("p", ":")
            t = _ttype(tk)
            args.append((n, t))
            types[n] = t
        tk.expect("arrow")
        rtypes = []
        if tk.accept("p", "("):
            rtypes.append(_ttype(tk))
            while tk.accept("p", ","):
                rtypes.append(_ttype(tk))
            tk.expect("p", ")")
        else:
            rtypes.append(_ttype(tk))
        tk.expect("p", "{")
        ops = []
        while not (tk.peek() == ("ident", "return")):
            ops.append(_op(tk, types, mesh))
        tk.expect("ident", "return")
        results = [_var(tk)]
        while tk.accept("p", ","):
            results.append(_var(tk))
        tk.expect("p", "}")
        if len(results) != len(rtypes) or any(types[r] != t for r, t in zip(results, rtypes)):
            raise ParseError(f"@{fname}: return does not match signature")
        funcs.append(Func(fname, args, ops, results, rtypes))
    return Module(funcs, mesh)


def collective_counts(module) -> dict:
    """Counted collectives (spmd.py:264-271; all_slice is free and absent)."""
    counts = {k: 0 for k in COUNTED_COLLECTIVES}
    for f in module.funcs:
        for op in f.ops:
            if op.kind in counts:
                counts[op.kind] += 1
    return counts


def op_flops(op, operand_dims) -> float:
    """FLOP convention of the reference simulator (sim.py:86-100)."""
    k = op.kind
    if k == "matmul":
        m, kk = operand_dims[0]
        return 2.0 * m * kk * operand_dims[1][1]
    if k in ("add", "mul", "neg", "exp"):
        return float(_prod(op.result_types[0].dims))
    if k == "reduce":
        return float(_prod(operand_dims[0]))
    return 0.0


def compute_flops(module, func: str = "main") -> float:
    """Per-device FLOPs as `simulate(...).compute_flops` counts them (sim.py:209-229)."""
    f = module.func(func)
    types = {n: t for n, t in f.args}
    total = 0.0
    for op in f.ops:
        for r, t in zip(op.results, op.result_types):
            types[r] = t
        if op.kind in COLLECTIVE_KINDS:
            continue
        total += op_flops(op, [types[o].dims for o in op.operands])
    return total
