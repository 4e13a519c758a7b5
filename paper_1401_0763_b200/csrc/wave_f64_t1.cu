// wave_f64_t1.cu — wave_kernel<double, T=1, LINK=false> and its launcher (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave_T<double, 1, 0, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 1, 1, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_T<double, 1, 2, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave_persist<double, 1>(sor_grid*, const Slab&, double, int, unsigned*);
}  // namespace sorh
