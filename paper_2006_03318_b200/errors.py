"""Error taxonomy of the simulator.

The class names and their ``.name`` strings are the stable identifiers of the
reference (pkg/src/kernsim/errors.py:11-140): CLI and HTTP callers match on
them, and the C-ABI maps its status codes onto them (include/ddsim.h).  The
classes are generated from a table rather than written out one by one.
"""

from __future__ import annotations


class KernsimError(Exception):
    """Root of the hierarchy; ``name`` is machine readable."""

    name = "KernsimError"

    def __init__(self, message: str = ""):
        super().__init__(message)
        self.message = message

    def __str__(self) -> str:
        if not self.message:
            return self.name
        return f"{self.name}: {self.message}"


class OverlapViolation(KernsimError):
    name = "OverlapViolation"

    def __init__(self, message: str, first_id: int, second_id: int):
        super().__init__(message)
        self.first_id = first_id
        self.second_id = second_id


class CycleDetected(KernsimError):
    name = "CycleDetected"

    def __init__(self, message: str, cycle: list[int] | None = None):
        super().__init__(message)
        self.cycle = list(cycle or [])


# Plain subclasses: (group, names).  Groups only document where each is raised.
_SIMPLE = {
    "trace": ("MalformedDocument", "SchemaViolation", "InvalidSpec", "MismatchedInput"),
    "graph": ("OrphanKernel",),
    "layers": ("AmbiguousMarker",),
    "comm": ("InvalidGroup", "MissingLayer", "NoWeightUpdate"),
    "sim": ("Deadlock", "ZeroBaseline"),
    "transform": ("WouldCreateCycle", "UnknownAnchor", "UnknownTask", "AcyclicityViolated",
                  "BadSelector", "BadPipeline"),
    "scenarios": ("BadFactorization", "MissingLayerGradients", "MissingConvPairs", "BadRatio",
                  "UnknownScenario"),
    # device boundary (include/ddsim.h status codes without a reference twin)
    "device": ("NoDevice", "CudaError", "OutOfMemory", "Unsupported", "UnsupportedPolicy"),
}

for _names in _SIMPLE.values():
    for _n in _names:
        globals()[_n] = type(_n, (KernsimError,), {"name": _n, "__module__": __name__})
del _names, _n

# Static names for linters / importers.
MalformedDocument = globals()["MalformedDocument"]
SchemaViolation = globals()["SchemaViolation"]
InvalidSpec = globals()["InvalidSpec"]
MismatchedInput = globals()["MismatchedInput"]
OrphanKernel = globals()["OrphanKernel"]
AmbiguousMarker = globals()["AmbiguousMarker"]
InvalidGroup = globals()["InvalidGroup"]
MissingLayer = globals()["MissingLayer"]
NoWeightUpdate = globals()["NoWeightUpdate"]
Deadlock = globals()["Deadlock"]
ZeroBaseline = globals()["ZeroBaseline"]
WouldCreateCycle = globals()["WouldCreateCycle"]
UnknownAnchor = globals()["UnknownAnchor"]
UnknownTask = globals()["UnknownTask"]
AcyclicityViolated = globals()["AcyclicityViolated"]
BadSelector = globals()["BadSelector"]
BadPipeline = globals()["BadPipeline"]
BadFactorization = globals()["BadFactorization"]
MissingLayerGradients = globals()["MissingLayerGradients"]
MissingConvPairs = globals()["MissingConvPairs"]
BadRatio = globals()["BadRatio"]
UnknownScenario = globals()["UnknownScenario"]
NoDevice = globals()["NoDevice"]
CudaError = globals()["CudaError"]
OutOfMemory = globals()["OutOfMemory"]
Unsupported = globals()["Unsupported"]
UnsupportedPolicy = globals()["UnsupportedPolicy"]
