"""Exception classes, named and typed as in the reference package.

segrender.py:39-48, distsim.py:63-64, partitioner.py:23-36.
"""


class VrError(RuntimeError):
    """A CUDA or library failure with no reference analogue."""


class CapacityError(VrError):
    """A kernel-side capacity bound was exceeded (bins per ray, segments per ray)."""


class GradientOverflowError(VrError):
    """A (scaled) MLP gradient is not representable in the tensor-core kernels' fp16
    operands (no reference analogue: the reference has no backward)."""


class NonFiniteInputError(ValueError):
    """A segment aggregate carries NaN or infinity (segrender.py:39-40)."""


class NegativeLossError(ValueError):
    """Composed distortion went negative beyond round-off (segrender.py:43-44)."""


class ParamNotOwnedError(KeyError):
    """The referenced parameter does not belong to the given region (segrender.py:47-48)."""


class ProtocolMismatchError(RuntimeError):
    """Empty pool or inconsistent broadcast composition (distsim.py:63-64)."""


class DegenerateSplitError(ValueError):
    """All candidate planes fail to separate the points (partitioner.py:23-24)."""


class InsufficientPointsError(ValueError):
    """Too few points to build the requested number of tiles (partitioner.py:27-28)."""


class NoPointsError(ValueError):
    """Ray discretisation produced no points inside the root box (partitioner.py:31-32)."""


class OutOfBoundsError(ValueError):
    """Point lies outside the partition's root box (partitioner.py:35-36)."""
