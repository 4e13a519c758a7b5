// wave2_f32_t4.cu — skew-2 wave2_kernel<float, T=4> and its launcher (see wave2.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave2_T<float, 4, 0, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave2_T<float, 4, 1, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave2_T<float, 4, 2, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave2_T<float, 4, 3, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave2_T<float, 4, 4, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
}  // namespace sorh
