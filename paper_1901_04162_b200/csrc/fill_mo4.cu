// fill_mo4.cu -- the fill kernels for 4 outer point(s) per triangle
// (one translation unit per outer-point count: parallel compilation).
#include "fill_kernels.cuh"

namespace gk {
template int dispatch_mo<4>(gk_ctx*, const FillArgs&, gk_mode, int, int, int,
                              const gk_fill_options&);
}  // namespace gk
