// wave_f32_t4.cu — wave_kernel<float, T=4, LINK=false> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<float, 4, 0, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 4, 1, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 4, 2, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 4, 3, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 4, 4, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_persist<float, 4>(sor_grid*, const Slab&, float, int, unsigned*);
}  // namespace sorh
