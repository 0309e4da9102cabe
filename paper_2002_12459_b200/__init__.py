"""paper_2002_12459_b200 -- B200-native join-project engine (MMJoin hot path).

Drop-in for the reference package ``mmjoin``'s join-project path
(arXiv 2002.12459): same entry points and result formats, computed by
hand-written sm_100a CUDA kernels in ``_lib/libmmjoin_b200.so`` (C ABI:
``include/mmjoin_b200.h``).  There is no CPU fallback.
"""

from . import errors, optimizer, relation
from .errors import MatrixOverflowError, ParseError, PlanError, StarResourceError
from .optimizer import FULL_JOIN, PARTITIONED, ThresholdPlan, default_plan, gpu_plan
from .relation import IndexedRelation, Relation, build_indexed, semi_join_reduce, semi_join_reduce_many

__version__ = "0.1.0"


def __getattr__(name):
    # operator modules import torch lazily so the host data model stays usable
    # (and testable) on machines without a GPU
    import importlib
    if name in ("joinproject", "matmul", "apps", "engine", "device", "datagen", "ingest", "calibration", "bsi",
                "star", "shard"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
