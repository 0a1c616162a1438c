"""HTTP transport over the GPU command layer (mirrors winoconv/service)."""
from .app import create_app  # noqa: F401
