// Forwarding header: the reference include name (proj/include/wavepipe/gantt.hpp)
// maps onto the consolidated API in wavepipe/core.hpp.
#pragma once
#include "wavepipe/core.hpp"
