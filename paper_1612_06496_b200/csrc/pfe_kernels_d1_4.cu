// Kernel instantiations for embedding dimensions 1..4 (see pfe_launch_impl.cuh).
#include "pfe_launch_impl.cuh"

namespace pfe_host {
template LaunchTable make_table<1>();
template LaunchTable make_table<2>();
template LaunchTable make_table<3>();
template LaunchTable make_table<4>();
}  // namespace pfe_host
