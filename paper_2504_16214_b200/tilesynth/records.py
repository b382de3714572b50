"""Record types from field tables (the synthesizer's plain-data classes).

``record("Name", fields, doc, **members)`` builds a dataclass: a bare field name is required,
``(name, default)`` optional, ``(name, list)`` / ``(name, dict)`` an empty-container default;
``members`` become class attributes (methods, properties, ``__post_init__``)."""
from __future__ import annotations

from dataclasses import field, make_dataclass


def record(cls_name, fields, doc, frozen=False, module=__name__, **members):
    spec = []
    for f in fields:
        if isinstance(f, str):
            spec.append(f)
        elif f[1] in (list, dict):
            spec.append((f[0], object, field(default_factory=f[1])))
        else:
            spec.append((f[0], object, field(default=f[1])))
    return make_dataclass(cls_name, spec, frozen=frozen, namespace={"__doc__": doc, **members}, module=module)
