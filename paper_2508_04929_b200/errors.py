"""Reference-compatible module path for the exception types (cryosplat.errors)."""
from .exceptions import *  # noqa: F401,F403
from .exceptions import __all__  # noqa: F401
