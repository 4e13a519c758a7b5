// wave2_f64_t5.cu — skew-2 wave2_kernel<double, T=5> and its launcher (see wave2.cuh); T > 4
// runs on single-slab handles only (no halo-pushing instance).
#include "wave_launch.cuh"

namespace sorh {
template int launch_wave2_T<double, 5, 0, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave2_T<double, 5, 1, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave2_T<double, 5, 2, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave2_T<double, 5, 3, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
template int launch_wave2_T<double, 5, 4, false>(sor_grid*, const Slab&, double, const IterCtl&, bool);
}  // namespace sorh
