// Kernel instantiations for embedding dimensions 5..8 (see pfe_launch_impl.cuh).
#include "pfe_launch_impl.cuh"

namespace pfe_host {
template LaunchTable make_table<5>();
template LaunchTable make_table<6>();
template LaunchTable make_table<7>();
template LaunchTable make_table<8>();
}  // namespace pfe_host
