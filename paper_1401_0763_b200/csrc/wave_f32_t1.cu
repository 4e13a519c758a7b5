// wave_f32_t1.cu — wave_kernel<float, T=1, LINK=false> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<float, 1, 0, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 1, 1, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 1, 2, false>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_persist<float, 1>(sor_grid*, const Slab&, float, int, unsigned*);
}  // namespace sorh
