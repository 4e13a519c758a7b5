// wave_f32_t1_link.cu — wave_kernel<float, T=1, LINK=true> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<float, 1, 0, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 1, 1, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 1, 2, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
}  // namespace sorh
