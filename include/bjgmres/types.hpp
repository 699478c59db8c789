// Forwarding header: keeps the reference's #include "bjgmres/types.hpp"
// (proj/include/bjgmres/types.hpp) valid; everything lives in bjgmres_b200.hpp.
#pragma once
#include "../bjgmres_b200.hpp"
