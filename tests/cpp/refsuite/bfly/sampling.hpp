// Include shim: the reference header bfly/sampling.hpp (reference proj/include/bfly/sampling.hpp)
// maps onto the B200 facade, which declares the same names in namespace bfly.
#pragma once
#include "bfly_b200.hpp"
