// Forwarding header: keeps the reference's #include "bjgmres/matrix_market.hpp"
// (proj/include/bjgmres/matrix_market.hpp) valid; everything lives in bjgmres_b200.hpp.
#pragma once
#include "../bjgmres_b200.hpp"
