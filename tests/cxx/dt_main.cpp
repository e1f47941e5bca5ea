#define DT_MAIN
#include "doctest.h"
