// Drop-in module header: the B200 implementation of the reference's
// spardl/collectives.hpp lives in spardl_b200.hpp (one header over the C ABI).
#pragma once
#include "spardl/spardl_b200.hpp"
