// Kernel instantiations for embedding dimensions 9..12 (see pfe_launch_impl.cuh).
#include "pfe_launch_impl.cuh"

namespace pfe_host {
template LaunchTable make_table<9>();
template LaunchTable make_table<10>();
template LaunchTable make_table<11>();
template LaunchTable make_table<12>();
}  // namespace pfe_host
