// jacobi_inst.cu — jacobi_kernel (NEXT-2) instances and launchers, LINK=false (see wave_launch.cuh).
#include "wave_launch.cuh"

namespace sorh {
template int launch_jacobi_T<double, 1, 0, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<double, 1, 1, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<double, 1, 2, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<double, 2, 0, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<double, 2, 1, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<double, 2, 2, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<double, 3, 0, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<double, 3, 1, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<double, 3, 2, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<double, 4, 0, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<double, 4, 1, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<double, 4, 2, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<float, 1, 0, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<float, 1, 1, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<float, 1, 2, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<float, 2, 0, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<float, 2, 1, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<float, 2, 2, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<float, 3, 0, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<float, 3, 1, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<float, 3, 2, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<float, 4, 0, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<float, 4, 1, false>(sor_grid*, const Slab&, const IterCtl&, bool);
template int launch_jacobi_T<float, 4, 2, false>(sor_grid*, const Slab&, const IterCtl&, bool);
}  // namespace sorh
