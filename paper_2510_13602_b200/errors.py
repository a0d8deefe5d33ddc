"""Exception types of the block manager, same names and hierarchy as the reference
(kv_manager.py:31-56) so callers' except-clauses keep working."""


class ManagerError(Exception):
    pass


class OutOfBlocks(ManagerError):
    pass


class DuplicateKey(ManagerError):
    pass


class UnknownKey(ManagerError):
    pass


class CapacityExceeded(ManagerError):
    pass


class StalePlan(ManagerError):
    pass


class LayoutMismatch(ManagerError):
    pass
