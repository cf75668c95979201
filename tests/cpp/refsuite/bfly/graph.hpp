// Include shim: the reference header bfly/graph.hpp (reference proj/include/bfly/graph.hpp)
// maps onto the B200 facade, which declares the same names in namespace bfly.
#pragma once
#include "bfly_b200.hpp"
