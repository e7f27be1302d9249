"""Exception classes of the reference, raised by the B200 host path.

Same names and base classes as reference tensor.py:20-25 (DimensionError,
NonFiniteError), model.py:28-33 (PartitionError, ScheduleViolation) and
engine.py:138-139 (WorkerFailure), so callers' `except` clauses carry over.
"""


class DimensionError(ValueError):
    """Operand shapes do not satisfy the operation's contract."""


class NonFiniteError(ArithmeticError):
    """A NaN or Inf appeared where only finite values are allowed."""


class PartitionError(ValueError):
    pass


class ScheduleViolation(RuntimeError):
    """A slot or snapshot queue was used outside the schedule's bounds."""


class WorkerFailure(RuntimeError):
    pass


class DeviceError(RuntimeError):
    """CUDA or NCCL failure reported by the native library."""


_STATUS = {
    1: DimensionError,
    2: NonFiniteError,
    3: ScheduleViolation,
    4: PartitionError,
    5: DeviceError,
    6: DeviceError,
    7: ValueError,
}


def raise_for_status(status, message):
    raise _STATUS.get(status, DeviceError)(message)
