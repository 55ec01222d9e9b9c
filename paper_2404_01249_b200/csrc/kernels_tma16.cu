// kernels_tma16.cu — the plane-streaming kernels of kernels_tma.cu instantiated
// with 16-wide x tiles (namespace dfm::tx16): kernels_tma.cu's public launchers
// pick them for mid-size levels whose last 32-wide tile would be at most half
// full (an 80-column level: 3 x 32 columns computed for 80, or 5 x 16).
#define DFM_TMA_TX 16
#define DFM_TMA_NS tx16
#define DFM_TMA_NO_DISPATCH
#include "kernels_tma.cu"
