// wave_f64_t3.cu — wave_kernel<double, T=3, LINK=false> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<double, 3, 0, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 3, 1, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 3, 2, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 3, 3, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 3, 4, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_persist<double, 3>(sor_grid*, const Slab&, double, int, unsigned*);
}  // namespace sorh
