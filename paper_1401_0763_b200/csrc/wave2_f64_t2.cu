// wave2_f64_t2.cu — skew-2 wave2_kernel<double, T=2> and its launcher (see wave2.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave2_T<double, 2, 0, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave2_T<double, 2, 1, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave2_T<double, 2, 2, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave2_T<double, 2, 3, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave2_T<double, 2, 4, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
}  // namespace sorh
