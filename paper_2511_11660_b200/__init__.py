"""B200-native (sm_100a) graph-based STA hot path of HeteroSTA (arxiv 2511.11660).

The product is libsta.so (include/sta.h); `sta` is its thin ctypes binding.
"""
from . import sta  # noqa: F401
from .sta import Context, StaError, load_design  # noqa: F401
