// wave_f64_t2.cu — wave_kernel<double, T=2, LINK=false> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<double, 2, 0, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 2, 1, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 2, 2, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 2, 3, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 2, 4, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_persist<double, 2>(sor_grid*, const Slab&, double, int, unsigned*);
}  // namespace sorh
