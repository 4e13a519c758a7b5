// wave2_f64_t3.cu — skew-2 wave2_kernel<double, T=3> and its launcher (see wave2.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave2_T<double, 3, 0, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave2_T<double, 3, 1, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave2_T<double, 3, 2, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave2_T<double, 3, 3, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave2_T<double, 3, 4, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
}  // namespace sorh
