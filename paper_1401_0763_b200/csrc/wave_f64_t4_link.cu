// wave_f64_t4_link.cu — wave_kernel<double, T=4, LINK=true> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<double, 4, 0, true>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 4, 1, true>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 4, 2, true>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 4, 3, true>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 4, 4, true>(sor_grid*, const Slab&, double, const IterCtl&, bool);
}  // namespace sorh
