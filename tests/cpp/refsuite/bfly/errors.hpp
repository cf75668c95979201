// Include shim: the reference header bfly/errors.hpp (reference proj/include/bfly/errors.hpp)
// maps onto the B200 facade, which declares the same names in namespace bfly.
#pragma once
#include "bfly_b200.hpp"
