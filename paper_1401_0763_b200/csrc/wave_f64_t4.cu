// wave_f64_t4.cu — wave_kernel<double, T=4, LINK=false> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<double, 4, 0, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 4, 1, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 4, 2, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 4, 3, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 4, 4, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_persist<double, 4>(sor_grid*, const Slab&, double, int, unsigned*);
}  // namespace sorh
