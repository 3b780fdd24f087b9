// Kernel instantiations for embedding dimensions 13..16 (see pfe_launch_impl.cuh).
#include "pfe_launch_impl.cuh"

namespace pfe_host {
template LaunchTable make_table<13>();
template LaunchTable make_table<14>();
template LaunchTable make_table<15>();
template LaunchTable make_table<16>();
}  // namespace pfe_host
