// Forwarding header: keeps the reference's #include "bjgmres/spmv.hpp"
// (proj/include/bjgmres/spmv.hpp) valid; everything lives in bjgmres_b200.hpp.
#pragma once
#include "../bjgmres_b200.hpp"
