// wave_f32_t4_link.cu — wave_kernel<float, T=4, LINK=true> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<float, 4, 0, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 4, 1, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 4, 2, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 4, 3, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 4, 4, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
}  // namespace sorh
