"""Loader of the reference-generated golden vectors (tests/golden/)."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2407_18352_b200.directives import parse_directive, parse_functor_decl

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(None)
def meta() -> dict:
    return json.loads((GOLDEN / "golden.json").read_text())


@lru_cache(None)
def arrays():
    return dict(np.load(GOLDEN / "golden.npz"))


def functor(text):
    return parse_functor_decl(text) if not text.startswith("functor(") else parse_directive(text)


def target(text, env=None):
    return parse_directive(f"map(to: f({text}))", env).targets[0]


def case(kind: str, i: int):
    c = meta()[kind][i]
    return functor(c["functor"]), target(c["target"]), c


def infer_layers(name):
    a = arrays()
    info = next(m for m in meta()["infer"] if m["name"] == name)
    layers = [(a[f"inf_{name}_W{k}"], a[f"inf_{name}_b{k}"], act)
              for k, act in enumerate(info["acts"])]
    return layers, a[f"inf_{name}_x"], a[f"inf_{name}_y"]
