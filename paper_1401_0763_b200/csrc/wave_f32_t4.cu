// wave_f32_t4.cu — wave_kernel<float, T=4> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<float, 4, 0>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 4, 1>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 4, 2>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 4, 3>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 4, 4>(sor_grid*, const Slab&, float, const IterCtl&, bool);
}  // namespace sorh
