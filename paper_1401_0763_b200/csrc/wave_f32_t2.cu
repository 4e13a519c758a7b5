// wave_f32_t2.cu — wave_kernel<float, T=2> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<float, 2, 0>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 2, 1>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 2, 2>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 2, 3>(sor_grid*, const Slab&, float, const IterCtl&, bool);
template int launch_wave_T<float, 2, 4>(sor_grid*, const Slab&, float, const IterCtl&, bool);
}  // namespace sorh
