"""Directive front end: the reference's criterion-7 corpus (test_acceptance.py:222-300)
and parse/print round trips."""

import random

import pytest

from paper_2407_18352_b200.directives import (ConcreteSlice, FunctorDecl, MapDirective, MapTarget,
                                              MlDirective, SliceDim, SymbolicSlice, SymExpr,
                                              parse_directive, parse_directive_file,
                                              parse_functor_decl, pretty_print)
from paper_2407_18352_b200.errors import (DirectiveSyntaxError, EmptyRangeError, MissingClauseError,
                                          SemanticError, UnboundVariableError,
                                          UnsupportedConstructError)

CORPUS = [
    "#pragma approx tensor functor(ifnctr: [i, j, 0:5] = ( ([i-1, j], [i+1, j], [i, j-1:j+2])))",
    "#pragma approx tensor functor(ofnctr: [i, j, 0:1] = ([i, j]))",
    "#pragma approx tensor map(to: ifnctr(t[1:N-1, 1:M-1]))",
    "#pragma approx tensor map(from: ofnctr(tnew[1:N-1, 1:M-1]))",
    '#pragma approx ml(predicated:true) in(t) out(tnew) db("/path/data.srdb") model("/path/model")',
    "f1: [i, 0:1] = ([i])", "functor(f2: [i, 0:2] = ([i-2], [i+2]))",
    "f3: [i, j, k, 0:3] = ([i, j, k-1:k+2])", "f4: [i, 0:4] = ([i-2:i+2])",
    "f5: [i, 0:2] = ([i-1:i+2:2])", "f6: [i, 0:3, j] = ([i, j-1:j+2])",
    "f7: [k, 0:5] = ([k, 0:5])", "f8: [k, 0:6] = ([k, 0:6:1])",
    "f9: [i, j, 0:2, 0:2] = ([i-1:i+1, j-1:j+1])", "f10: [i, 0:2] = ([i], [i+1])",
    "map(to: f1(a[0:16]))", "map(to: f3(v[1:7, 1:7, 1:7]))", "map(from: f1(b[2:10:2]))",
    "map(to: f7(recs[0:COUNT]))", "map(to: f1(a[0:8], b[0:8]))", "tensor map(to: f1(a[3:5]))",
    'ml(infer) in(a) out(b) model("m")', 'ml(collect) in(a) out(b) db("d.srdb")',
    'ml(collect) inout(state) database("d.srdb")',
    'ml(predicated:step % 2 == 0) in(a) out(b) db("d") model("m")',
    'ml(infer) in(a, b) out(c) model("m") if(enabled && step > 10)',
]
ENV = {"N": 16, "M": 16, "COUNT": 1024}


def test_corpus_parses_and_round_trips():
    asts = [parse_directive(t, ENV) for t in CORPUS]
    assert sum(isinstance(a, FunctorDecl) for a in asts) == 12
    assert {a.direction for a in asts if isinstance(a, MapDirective)} == {"to", "from"}
    assert {a.mode for a in asts if isinstance(a, MlDirective)} == {"infer", "collect", "predicated"}
    for a in asts:
        assert parse_directive(pretty_print(a), ENV) == a


def test_stencil_functor_fields():
    f = parse_directive(CORPUS[0])
    assert f.symbols == ("i", "j") and f.feature_sizes == (5,)
    assert f.rhs[2].dims[1] == SliceDim(SymExpr("j", -1), SymExpr("j", 2), 1)
    m = parse_directive(CORPUS[2], {"N": 4, "M": 4})
    assert m.targets[0] == MapTarget("t", (ConcreteSlice(1, 3), ConcreteSlice(1, 3)))
    ml = parse_directive(CORPUS[4])
    assert ml.predicate == "true" and ml.model_path == "/path/model" and ml.db_path == "/path/data.srdb"
    ml = parse_directive(CORPUS[-1])
    assert ml.if_cond == "enabled && step > 10" and ml.in_refs == ("a", "b")


def test_directive_file_offsets():
    text = ("#pragma approx tensor functor(ifnctr: \\\n    [i, j,  0:5] = ( ([i-1, j], [i+1, j], \\\n"
            "    [i, j-1:j+2])))\n// comment line\n\n#pragma approx tensor map(to: \\\n"
            "    ifnctr(t[1:N-1, 1:M-1]))\n")
    asts = parse_directive_file(text, {"N": 4, "M": 4})
    assert len(asts) == 2 and asts[1].targets[0].slices[0] == ConcreteSlice(1, 3)
    bad = "f1: [i, 0:1] = ([i])\nf2: [i, 0:1] = ([i] $)\n"
    with pytest.raises(DirectiveSyntaxError) as e:
        parse_directive_file(bad)
    assert bad[e.value.offset] == "$"


@pytest.mark.parametrize("text,exc", [
    ("f: [i, 0:1] = ([i*2])", SemanticError),
    ("f: [i, 0:1] = ([i+j])", SemanticError),
    ("f: [i, 0:1] = ([j])", SemanticError),
    ("f: [i] = ([i])", SemanticError),
    ("f: [0:2] = ([0])", SemanticError),
    ("f: [i, 0:1] = ([i:j])", SemanticError),
    ("f: [i, 3:1] = ([i])", SemanticError),
    ("map(to: f(a[0:N]))", UnboundVariableError),
    ("map(to: f(a[4:2]))", EmptyRangeError),
    ("map(to: f(a[b[0:2]]))", UnsupportedConstructError),
    ("map(sideways: f(a[0:2]))", DirectiveSyntaxError),
    ('ml(infer) in(a) out(b)', MissingClauseError),
    ('ml(collect) out(b) db("d")', MissingClauseError),
    ('ml(infer) in(a) out(b) model("m") model("n")', DirectiveSyntaxError),
    ('ml(guess) in(a) out(b)', DirectiveSyntaxError),
    ('ml(infer) in(a) out(b) model("m', DirectiveSyntaxError),
    ('ml(infer:(x) in(a)', DirectiveSyntaxError),
])
def test_errors(text, exc):
    with pytest.raises(exc):
        parse_directive(text)


def _rand_functor(rng):
    syms = list(dict.fromkeys(rng.choice("ijkpq") for _ in range(rng.randint(1, 3))))
    lhs = [SliceDim(SymExpr.sym(s)) for s in syms]
    for _ in range(rng.randint(1, 2)):
        lo = rng.randint(0, 3)
        d = SliceDim(SymExpr.const(lo), SymExpr.const(lo + rng.randint(1, 6)), rng.choice([1, 2]))
        lhs.insert(rng.randrange(len(lhs) + 1), d)
    rhs = []
    for _ in range(rng.randint(1, 3)):
        dims = []
        for s in syms:
            if rng.random() < 0.3:
                lo = rng.randint(-2, 0)
                dims.append(SliceDim(SymExpr.sym(s, lo), SymExpr.sym(s, lo + rng.randint(1, 3)),
                                     rng.choice([1, 2])))
            else:
                dims.append(SliceDim(SymExpr.sym(s, rng.randint(-3, 3))))
        if rng.random() < 0.2:
            lo = rng.randint(0, 4)
            dims.append(SliceDim(SymExpr.const(lo), SymExpr.const(lo + rng.randint(1, 4))))
        rhs.append(SymbolicSlice(tuple(dims)))
    return FunctorDecl(rng.choice(["fn", "g_2", "probe"]), SymbolicSlice(tuple(lhs)), tuple(rhs))


def _rand_ast(rng):
    r = rng.random()
    if r < 0.4:
        return _rand_functor(rng)
    if r < 0.7:
        ts = tuple(MapTarget(rng.choice(["t", "tnew", "recs"]),
                             tuple(ConcreteSlice(a, a + rng.randint(1, 12), rng.choice([1, 2, 3]))
                                   for a in [rng.randint(0, 8) for _ in range(rng.randint(1, 3))]))
                   for _ in range(rng.randint(1, 2)))
        return MapDirective(rng.choice(["to", "from"]), "fn", ts)
    mode = rng.choice(["infer", "collect", "predicated"])
    return MlDirective(mode, predicate="use_nn" if mode == "predicated" else None,
                       in_refs=("a",), out_refs=("b", "c")[: rng.randint(1, 2)],
                       model_path="m/x" if mode != "collect" else None,
                       db_path="d.srdb" if mode != "infer" else None,
                       if_cond=rng.choice([None, "step > 100"]))


def test_random_round_trips():
    rng = random.Random(0xC0FFEE)
    for _ in range(200):
        ast = _rand_ast(rng)
        once = pretty_print(ast)
        assert pretty_print(parse_directive(once)) == once
        assert parse_directive(once) == ast
