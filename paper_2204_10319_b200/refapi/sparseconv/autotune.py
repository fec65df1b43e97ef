"""``sparseconv.autotune`` on the B200 engine: the reference's search API
and JSON v1 strategy files (reference ``autotune.py``) with device cost
models.  This name IS the engine module (:mod:`paper_2204_10319_b200.autotune`),
so patching ``sparseconv.autotune.<name>`` patches what the engine uses, as
patching the reference's module does there."""

import sys

from paper_2204_10319_b200 import autotune as _engine

sys.modules[__name__] = _engine
