// wave_f32_t3.cu — wave_kernel<float, T=3, LINK=false> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<float, 3, 0, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 3, 1, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 3, 2, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 3, 3, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 3, 4, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_persist<float, 3>(sor_grid*, const Slab&, float, int, unsigned*);
}  // namespace sorh
