// Forwarding header: keeps the reference's #include "bjgmres/sparse_matrix.hpp"
// (proj/include/bjgmres/sparse_matrix.hpp) valid; everything lives in bjgmres_b200.hpp.
#pragma once
#include "../bjgmres_b200.hpp"
