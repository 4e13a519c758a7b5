// wave2_f32_t6.cu — skew-2 wave2_kernel<float, T=6> and its launcher (see wave2.cuh); T > 4
// runs on single-slab handles only (no halo-pushing instance).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave2_T<float, 6, 0, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave2_T<float, 6, 1, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave2_T<float, 6, 2, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave2_T<float, 6, 3, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave2_T<float, 6, 4, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
}  // namespace sorh
