"""Error types mirroring the reference (errors.py:4-13)."""


class FormatError(ValueError):
    """A model / field file is malformed."""


class SceneValidationError(ValueError):
    """A scene description violates an invariant."""
