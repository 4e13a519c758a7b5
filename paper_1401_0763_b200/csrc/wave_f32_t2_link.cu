// wave_f32_t2_link.cu — wave_kernel<float, T=2, LINK=true> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<float, 2, 0, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 2, 1, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 2, 2, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 2, 3, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 2, 4, true>(sor_grid*, const Slab&, float, const IterCtl&, bool);
}  // namespace sorh
