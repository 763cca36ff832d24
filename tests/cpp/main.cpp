#include "doctest.h"

int main() { return mini_doctest::run_all(); }
