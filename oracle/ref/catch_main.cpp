// catch_main.cpp -- ORACLE (test infrastructure): test runner for the shimmed Catch2.
#include <catch2/catch_amalgamated.hpp>
int main() { return Catch::run_all(); }
