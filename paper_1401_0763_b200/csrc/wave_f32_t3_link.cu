// wave_f32_t3_link.cu — wave_kernel<float, T=3, LINK=true> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<float, 3, 0, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 3, 1, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 3, 2, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 3, 3, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 3, 4, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
}  // namespace sorh
