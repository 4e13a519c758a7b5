// wave_f64_t3_link.cu — wave_kernel<double, T=3, LINK=true> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<double, 3, 0, true>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 3, 1, true>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 3, 2, true>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 3, 3, true>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 3, 4, true>(sor_grid*, const Slab&, double, const IterCtl&, bool);
}  // namespace sorh
