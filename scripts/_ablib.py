"""A/B helper for the scripts (never the product path): TOKENRING_LIB=<path>
points this script's process at another build of libtokenring (a variant or
the experiments build) through ``_lib.use_library``."""
import os


def maybe_use_env_library():
    path = os.environ.get("TOKENRING_LIB")
    if path:
        from paper_2412_20501_b200 import _lib
        _lib.use_library(path)
        return path
    return None
