// Forwarding header: keeps the reference's #include "bjgmres/graph.hpp"
// (proj/include/bjgmres/graph.hpp) valid; everything lives in bjgmres_b200.hpp.
#pragma once
#include "../bjgmres_b200.hpp"
