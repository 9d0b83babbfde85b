"""B200-native (sm_100a) XQuant decode hot path (arxiv 2508.10395).

Drop-in for the reference package ``xcache``'s kernel lane
(``kernels``), cache backends (``cache``) and decode driver (``decode``).
The compute runs in the C-ABI library ``libxquant.so`` (include/xquant.h);
there is no CPU fallback.
"""

__version__ = "0.1.0"
