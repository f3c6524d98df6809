"""Drop-in shim: `import moepack` resolves to this repo's package, so the
REFERENCE's own test modules (tests/test_codec.py,
test_dictionary.py, ...) run unmodified against the GPU implementation.
Used only by tools/reference_tests.sh; not part of the product."""

import importlib
import sys

import paper_2310_16795_b200 as _q

for _name in ("bf16", "cli", "codec", "dictionary", "errors", "pipeline", "quantize", "stats"):
    sys.modules[f"moepack.{_name}"] = importlib.import_module(f"paper_2310_16795_b200.{_name}")

from paper_2310_16795_b200 import *  # noqa: E402,F401,F403

__version__ = _q.__dict__.get("__version__", "drop-in")
