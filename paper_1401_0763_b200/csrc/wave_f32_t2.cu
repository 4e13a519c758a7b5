// wave_f32_t2.cu — wave_kernel<float, T=2, LINK=false> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<float, 2, 0, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 2, 1, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 2, 2, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 2, 3, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 2, 4, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_persist<float, 2>(sor_grid*, const Slab&, float, int, unsigned*);
}  // namespace sorh
