// wave2_f32_t2.cu — skew-2 wave2_kernel<float, T=2> and its launcher (see wave2.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave2_T<float, 2, 0, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave2_T<float, 2, 1, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave2_T<float, 2, 2, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave2_T<float, 2, 3, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave2_T<float, 2, 4, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
}  // namespace sorh
